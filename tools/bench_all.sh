#!/bin/bash
# Developer driver (run on the GPU box from the repo root): every bench
# workload's JSON line into gpurun_out/bench_all.jsonl, the reference arm,
# the ncu launch list of the default bench and full captures of the default
# kernel and of the SIP wavefront kernel.  Numbers printed under ncu are not
# bench values.
set -u
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/bench_all.jsonl
run() { timeout 600 python bench.py "$@" 2> $OUT/bench_err.log | tail -1 >> $OUT/bench_all.jsonl; }
run --steps 20 --warmup 5
run --workload ntdm --steps 30 --warmup 5   # (a 23-us step: 5 steps are noise)
for w in mnpdm ntdm8k sip stdm spdm hb adi; do run --workload $w --steps 5 --warmup 3; done
run --workload npdm --algo sequential --steps 5 --warmup 3
run --impl reference --steps 3 --warmup 3
run --workload sip --sip-algo wavefront --steps 5 --warmup 3
run --impl reference --workload sip --steps 2 --warmup 3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_npdm.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:halo_kernel -s 3 -c 1 \
  -o $OUT/npdm_full python tools/sweep_part.py child 2 4096 8192 > $OUT/ncu_npdm.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sip_wave -s 1 -c 1 \
  -o $OUT/sip_full python bench.py --workload sip --sip-algo wavefront --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_sip.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sip_scan -s 1 -c 1 \
  -o $OUT/sip_scan_full python bench.py --workload sip --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_sip_scan.log 2>&1
echo done

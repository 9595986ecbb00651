# Developer A/B (GPU box): sparse-outer MNPDM bench line for library variants
set -u
run() { echo "== $1"; BX_LIB=$2 python bench.py --workload mnpdm --steps 10 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"; }
run base paper_1804_09666_b200/libbandix_b200.so
for v in "$@"; do
  d=/tmp/v_$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  python tools/variant_lib.py $d $v > /dev/null 2>&1; run "$v" $d/libbandix_b200.so
done

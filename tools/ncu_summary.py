"""Summarise an `ncu --set full` report into profiles/ (text) and record the
kernel's DRAM traffic per launch in profiles/traffic.json (read by bench.py
for roofline.traffic).

    python tools/ncu_summary.py REPORT.ncu-rep WORKLOAD OUT.txt [--note TEXT]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warp_latency_issue_stalled_barrier",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}, hdr, vals


def main():
    report, workload, out = sys.argv[1:4]
    note = sys.argv[sys.argv.index("--note") + 1] if "--note" in sys.argv else ""
    d, hdr, vals = raw(report)
    name = d.get("Kernel Name", ("?", ""))[0]

    def num(k):
        v, u = d[k]
        v = float(v.replace(",", ""))
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "nsecond": 1e-9,
                 "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6,
                 "ms": 1e-3, "s": 1}
        return v * scale.get(u, 1)
    lines = [f"report: {os.path.basename(report)}", f"kernel: {name}", f"workload: {workload}"]
    if note:
        lines.append(f"note: {note}")
    for k in KEYS:
        if k in d:
            lines.append(f"{k:70s} {d[k][0]:>16s} {d[k][1]}")
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    t = num("gpu__time_duration.sum")
    lines.append(f"dram bytes per launch (read+write) = {rd + wr:.6e}  -> {(rd + wr) / t / 1e9:.1f} GB/s "
                 f"over the ncu-timed launch (serialised, cold cache)")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(os.path.dirname(out), "traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    tj[workload] = {"bytes_per_launch": rd + wr, "read": rd, "write": wr,
                    "source": f"profiles/{os.path.basename(out)} (ncu --set full, {os.path.basename(report)})"}
    json.dump(tj, open(tp, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()

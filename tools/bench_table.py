"""Developer tool: format the JSON lines of tools/bench_all.sh into the
markdown table kept under profiles/ (every bench line of the round).

    python tools/bench_table.py gpurun_out/bench_all.jsonl profiles/r1_bench_lines.md
"""
import json
import sys

src, out = sys.argv[1], sys.argv[2]
rows, raw = [], []
for line in open(src):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    raw.append(line)
    rf = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    wl = d["config"].get("workload", "")
    algo = d["config"].get("algo", "")
    name = ("reference arm: " if d.get("impl") == "reference" else "") + wl + (f" [{algo}]" if algo else "")
    frac = f"{rf['frac']:.3f} ({rf['achieved']:.1f}/{rf['peak']:.1f} {rf['unit']})" if rf else "-"
    rows.append(f"| {name} | {d['value']:.4g} | {d['unit']} | {d['ms_per_step']:.3f} | {frac} | "
                f"{e2e.get('value', float('nan')):.4g} | {e2e.get('pcie_frac', '-')} | "
                f"{cpu.get('value') if cpu else None} ({cpu.get('cores', '-')} cores) |")
with open(out, "w") as f:
    f.write("# Bench lines of the round (B200, 1 GPU; `tools/bench_all.sh`, driver-style JSON)\n\n")
    f.write("| workload | value | unit | ms/step | roofline frac (achieved/peak) | e2e (host buffers) "
            "| PCIe H2D frac | cpu_baseline (C port) |\n|---|---|---|---|---|---|---|---|\n")
    f.write("\n".join(rows) + "\n\nRaw JSON lines:\n\n")
    for r in raw:
        f.write("```json\n" + r + "\n```\n")
print(open(out).read()[:3000])

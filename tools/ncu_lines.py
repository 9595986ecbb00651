"""Developer tool: per-source-line warp-stall samples from an ncu report
(`ncu -i R --page source --csv --print-source cuda,sass`).

    python tools/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, lines, tot = "?", None, [], 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        sc = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        s, e = int(r[iS]), int(r[iE])
    except ValueError:
        continue
    st = {hdr[i][6:]: int(r[i]) for i in sc if r[i].isdigit() and int(r[i]) > 0}
    lines.append((s, fname, r[0], r[1].strip()[:64], e, st))
    tot += s
lines.sort(key=lambda x: -x[0])
print("total samples", tot)
for s, f, ln, src, e, st in lines[:top]:
    t3 = ",".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{s:7d} {100 * s / max(tot, 1):5.1f}% {f}:{ln:<4} inst={e:9d} {src:64s} {t3}")

if len(sys.argv) > 3:  # ranges "a-b,c-d" of lines of the first file: summed samples per range
    for rg in sys.argv[3].split(","):
        a, b = map(int, rg.split("-"))
        sel = [x for x in lines if x[2].isdigit() and a <= int(x[2]) <= b and x[1].endswith(".cu")]
        agg = {}
        for x in sel:
            for k, v in x[5].items():
                agg[k] = agg.get(k, 0) + v
        t3 = ",".join(f"{k}:{v}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:4])
        print(f"lines {rg:10s} samples {sum(x[0] for x in sel):7d} inst {sum(x[4] for x in sel):10d}  {t3}")

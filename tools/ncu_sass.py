"""Developer tool: top SASS instructions by warp-stall samples from an ncu
report, with the source line each maps to.

    python tools/ncu_sass.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
L = []
for idx, r in enumerate(rows[2:]):
    try:
        L.append((int(r[iS]), idx, r[1].strip(), int(r[iE]),
                  {hdr[i][6:]: int(r[i]) for i in sc if r[i].isdigit() and int(r[i]) > 0}))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in L)
print("total samples", tot, "instructions", len(L))
for s, idx, src, e, st in sorted(L, reverse=True)[:top]:
    t2 = ",".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:2])
    print(f"{s:6d} {100 * s / tot:5.1f}% #{idx:5d} {src[:58]:58s} n={e:9d} {t2}")
if len(sys.argv) > 3:
    for rg in sys.argv[3].split(","):
        a, b = map(int, rg.split("-"))
        sel = [x for x in L if a <= x[1] < b]
        print(f"#{rg:12s} samples {sum(x[0] for x in sel):7d} inst {sum(x[3] for x in sel):11d}")

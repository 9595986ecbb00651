# Developer tool: per-kernel durations (ncu launch list) of a command's last kernels
# usage: [FILTER=substr] bash tools/launch_list.sh N CMD...   (prints the last N launches whose name contains FILTER)
N=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file /tmp/ll.csv "$@" > /dev/null 2>&1
python - "$N" <<'PY'
import csv, sys
import os
rows = [r for r in csv.DictReader(l for l in open("/tmp/ll.csv") if not l.startswith("=="))
        if os.environ.get("FILTER", "") in r["Kernel Name"]]
for r in rows[-int(sys.argv[1]):]:
    print(r["Kernel Name"][:70], r["Metric Value"], r["Metric Unit"])
PY

# Developer tool: per-kernel durations of one partitioned solve (ncu launch list)
# usage: bash tools/launch_list.sh K N B
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file /tmp/ll.csv python tools/sweep_part.py child $1 $2 $3 > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.DictReader(l for l in open("/tmp/ll.csv") if not l.startswith("==")))
for r in rows[-8:]:
    print(r["Kernel Name"][:70], r["Metric Value"], r["Metric Unit"])
PY

#!/bin/bash
# per-kernel durations (ncu, serialized, cold) of a short bench run
# usage: profiles/launch_list.sh <tag> [bench args...]
tag=$1; shift
cmd="python bench.py --steps 3 --warmup 3 --sweep 0 --no-cpu-baseline $*"
$cmd > gpurun_out/plain_$tag.log 2>&1 || { tail -n 3 gpurun_out/plain_$tag.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv $cmd > /dev/null 2>&1
python - "$tag" <<'P'
import csv, collections, sys
rows = list(csv.reader(open(f"gpurun_out/launches_{sys.argv[1]}.csv")))
i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[i]; kn = h.index("Kernel Name"); mv = h.index("Metric Value")
t = collections.defaultdict(list)
for r in rows[i + 1:]:
    if len(r) > mv:
        t[r[kn].split("(")[0][:48]].append(float(r[mv].replace(",", "")) / 1e3)
for k, v in t.items():
    print(f"{sys.argv[1]:10s} {k:50s} n={len(v):3d} mean_us={sum(v)/len(v):9.2f}")
P

#!/bin/bash
# per-kernel launch list of the config-3-sized implicit path (bench.implicit_measure)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/implicit_launches.csv python -c "
import sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench; r = bench.implicit_measure(0, cpu=False)" > gpurun_out/implicit_ncu.log 2>&1
python - <<'P'
import csv, collections
rows = [r for r in csv.DictReader(l for l in open('gpurun_out/implicit_launches.csv') if l.startswith('"'))]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r['Metric Name'] != 'gpu__time_duration.sum': continue
    k = r['Kernel Name'].split('(')[0].split('<')[0]
    v = float(r['Metric Value']) * (1e-3 if r['Metric Unit'] in ('ns', 'nsecond') else 1.0)
    agg[k][0] += 1; agg[k][1] += v
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f'{k:40s} {n:7d} {t:10.1f} us {t/n:8.2f} us/launch')
P

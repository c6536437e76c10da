python -c "import __graft_entry__ as g; g.build()"
python tools/debug/config3_scan_probe.py
ST_NO_PDL=1 python tools/debug/config3_scan_probe.py
NSTEPS=512 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3scan_launches.csv python tools/debug/config3_scan_probe.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/c3scan_launches.csv')) if len(r)>5]
i=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); h=rows[i]
kn,mv=h.index('Kernel Name'),h.index('Metric Value')
from collections import defaultdict
t=defaultdict(list)
for r in rows[i+1:]: t[r[kn].split('(')[0]].append(float(r[mv].replace(',',''))/1e3)
for k,v in sorted(t.items(), key=lambda x:-sum(x[1])): print(f"{k[:60]:60s} n={len(v):6d} mean={sum(v)/len(v):8.2f} us total={sum(v)/1e3:8.2f} ms")
PY

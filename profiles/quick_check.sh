#!/bin/bash
# quick GPU check: gpu tests + bench (config 1 + config 2 sweep), one line per workload
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python bench.py --steps 50 --no-cpu-baseline --sweep 1 > gpurun_out/b.log 2>&1 || tail -20 gpurun_out/b.log
python - <<'P'
import json
d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('c1', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2))
for k,v in d.get('sweep_config2',{}).items(): print(k, round(v['ms_per_step'],3), round(v['value']/1e9,2))
P

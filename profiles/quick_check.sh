#!/bin/bash
# quick GPU check: gpu tests + bench (sweep)
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python bench.py --steps 50 --no-cpu-baseline --sweep 1 > gpurun_out/b.log 2>&1
python - <<'P'
import json
d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('c1', d['ms_per_step'], d['roofline']['kernel_ms'], d['value']/1e9)
for k,v in d.get('sweep_config2',{}).items(): print(k, v['ms_per_step'], round(v['value']/1e9,2))
P

#!/bin/bash
# A/B of the structured hot kernels (k_xmarch vs k_xslab) on GPU: tests + sweep
for kk in slab march; do
  echo "== ST_KERNEL=$kk"
  ST_KERNEL=$kk python -m pytest tests -m gpu -x -q > gpurun_out/t_$kk.log 2>&1; tail -2 gpurun_out/t_$kk.log
  ST_KERNEL=$kk python bench.py --steps 30 --no-cpu-baseline --sweep 1 > gpurun_out/b_$kk.log 2>&1
  python - "$kk" <<'P'
import json,sys
d=json.loads(open(f'gpurun_out/b_{sys.argv[1]}.log').read().strip().splitlines()[-1])
print('c1', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,2))
for k,v in d.get('sweep_config2',{}).items(): print(k, round(v['ms_per_step'],3), round(v['value']/1e9,2))
P
done

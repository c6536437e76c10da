#!/bin/bash
# A/B of kernel variants: profiles/ab.sh v1 v2 ... ("base" = default library)
for v in "$@"; do
  if [ "$v" = base ]; then unset ST_VARIANT; else export ST_VARIANT=$v; fi
  python bench.py --steps 50 --no-cpu-baseline --sweep ${SWEEP:-1} > gpurun_out/b_$v.log 2>&1 || tail -5 gpurun_out/b_$v.log
  python - "$v" <<'P'
import json,sys
d=json.loads(open(f'gpurun_out/b_{sys.argv[1]}.log').read().strip().splitlines()[-1])
s=' '.join(f"{k}:{v['ms_per_step']:.3f}" for k,v in d.get('sweep_config2',{}).items())
print(f"{sys.argv[1]:10s} c1 {d['ms_per_step']:.4f} kern {d['roofline']['kernel_ms']:.4f}  {s}")
P
done

#!/bin/bash
# A/B of programmatic dependent launch (ST_NO_PDL=1 = plain launches): headline, e2e, sweep, config-3 explicit
for z in 1 0 1 0; do
  ST_NO_PDL=$z python bench.py --steps 100 --no-cpu-baseline --sweep 1 > gpurun_out/b_pdl$z.log 2>&1 || tail -5 gpurun_out/b_pdl$z.log
  python - "$z" <<'P'
import json,sys
z=sys.argv[1]
d=json.loads(open(f'gpurun_out/b_pdl{z}.log').read().strip().splitlines()[-1])
s=' '.join(f"{k}:{v['ms_per_step']:.3f}" for k,v in d.get('sweep_config2',{}).items())
i=d['implicit_config3']
print(f"nopdl={z} c1 {d['ms_per_step']:.4f} kern {d['roofline']['kernel_ms']:.4f} e2e {d['e2e']['value']/1e9:.2f} {s} c3expl {i['explicit_us_per_step']:.2f} be {i['ms_per_be_step']:.3f} crit {i['step_criteria_ms']:.1f}")
P
done

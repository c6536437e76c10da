#!/bin/bash
# A/B of the PDL chains on the config-3-sized implicit / scan / step-criteria measurement (after the GPU tests)
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for z in 1 0 1 0; do
ST_NO_PDL=$z python -c "
import sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench; r = bench.implicit_measure(0, cpu=False); print('nopdl=$z', round(r['ms_per_be_step'],3), round(r['us_per_cg_iteration'],1), round(r['explicit_us_per_step'],2), round(r['step_criteria_ms'],2), r['power_iterations'], r['dt_stability'])"
done

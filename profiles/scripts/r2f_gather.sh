# staged condensed gather + one PCG block per SM: unstructured parity tests, PCG phase clocks (dev hook
# -DST_PCG_TIMING), config-3 timings
set -x
timeout 1200 python -m pytest tests/test_gpu_operator.py tests/test_gpu_config3.py tests/test_gpu_snapshot.py tests/test_gpu_schedule.py -q -x 2>&1 | tail -3
ST_VARIANT=pcgt python tools/time_implicit.py 20 2>&1 | tail -2
python tools/time_implicit.py 20 2>&1 | tail -1
ST_VARIANT=pcgt PYTHONPATH=. python tools/debug/imp_phases.py 2>&1 | tail -2
python - <<'P'
import json, bench
r = bench.implicit_measure(0, cpu=False)
print({k: r[k] for k in ("ms_per_be_step", "cg_per_step", "us_per_cg_iteration", "explicit_us_per_step", "pcg_solve")})
c = bench.config3_build_measure(cpu=False)
print("config3_build wall_s_per_layer", c["wall_s_per_layer"], [(l["wall_scan"], l["wall_cool"]) for l in c["per_layer"]])
P
python tools/debug/config3_scan_probe.py 2>&1 | tail -1

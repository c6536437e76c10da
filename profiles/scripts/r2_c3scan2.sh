python -c "import __graft_entry__ as g; g.build()"
python tools/debug/config3_scan_probe.py
timeout 900 python -m pytest tests/test_gpu_config3.py tests/test_gpu_operator.py tests/test_gpu_schedule.py -q 2>&1 | tail -2
python - <<'PY' 2>&1 | tail -2
import sys, json, time; sys.argv=['bench.py']
import bench
r = bench.implicit_measure(0, cpu=False)
print('be_ms %.4f pcg_us %.2f (it %d) expl_us %.2f crit_ms %.2f' % (r['ms_per_be_step'], r['pcg_solve']['us_per_iteration'], r['pcg_solve']['iterations'], r['explicit_us_per_step'], r['step_criteria_ms']))
r=bench.config3_build_measure(cpu=False); print(json.dumps({k:v for k,v in r.items() if k!='per_layer'}))
PY

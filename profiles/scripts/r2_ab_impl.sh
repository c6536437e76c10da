python -c "import __graft_entry__ as g; g.build()"
for cg in 0 1; do for sc in 0 1; do
ST_CG_PERSISTENT=$cg ST_SCAN_PERSISTENT=$sc python - <<'PY' 2>&1 | tail -1
import sys, json, os; sys.argv=['bench.py']
import bench
r = bench.implicit_measure(0, cpu=False)
print(os.environ['ST_CG_PERSISTENT'], os.environ['ST_SCAN_PERSISTENT'], 'be_ms %.4f pcg_us %.2f (it %d) expl_us %.2f crit_ms %.2f' % (r['ms_per_be_step'], r['pcg_solve']['us_per_iteration'], r['pcg_solve']['iterations'], r['explicit_us_per_step'], r['step_criteria_ms']))
PY
done; done

python -c "import __graft_entry__ as g; g.build()"
ST_VARIANT=minb1 ST_NVCC_EXTRA="-DST_PCG_MINB=1" python -m paper_2302_05164_b200._build > /dev/null
for v in "" minb1; do for cg in 0 1; do
ST_VARIANT=$v ST_CG_PERSISTENT=$cg python - <<'PY' 2>&1 | tail -1
import sys, json, os; sys.argv=['bench.py']
import bench
r = bench.implicit_measure(0, cpu=False)
print(repr(os.environ.get('ST_VARIANT')), os.environ['ST_CG_PERSISTENT'], 'be_ms %.4f pcg_us %.2f (it %d) expl_us %.2f' % (r['ms_per_be_step'], r['pcg_solve']['us_per_iteration'], r['pcg_solve']['iterations'], r['explicit_us_per_step']))
PY
done; done
timeout 900 python -m pytest tests/test_gpu_config3.py tests/test_gpu_operator.py -q -x 2>&1 | tail -2

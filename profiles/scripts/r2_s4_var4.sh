# (the ST_X2_INTERP_PLANES / ST_QP_REV hooks of this sweep were removed after the measurement: no gain)
python -c "import __graft_entry__ as g; g.build()" || exit 1
ST_VARIANT=ipl ST_NVCC_EXTRA="-DST_X2_INTERP_PLANES=1" python -m paper_2302_05164_b200._build > /dev/null
ST_VARIANT=qrev ST_NVCC_EXTRA="-DST_QP_REV=1" python -m paper_2302_05164_b200._build > /dev/null
ST_VARIANT=both ST_NVCC_EXTRA="-DST_QP_REV=1 -DST_X2_INTERP_PLANES=1" python -m paper_2302_05164_b200._build > /dev/null
timeout 300 python -m pytest tests/test_gpu_xmarch2.py -q -x 2>&1 | tail -2
ST_VARIANT=ipl timeout 300 python -m pytest tests/test_gpu_xmarch2.py -q -x 2>&1 | tail -2
for v in base ipl qrev both; do
if [ "$v" = base ]; then unset ST_VARIANT; else export ST_VARIANT=$v; fi
for wl in config4; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --sweep 0 --no-cpu-baseline > gpurun_out/var_${v}_$wl.json 2>gpurun_out/var_${v}_$wl.err; echo "$wl rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/var_${v}_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $wl', 'value %.4g ms %.4f kernel %.4f frac %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))"
done; done

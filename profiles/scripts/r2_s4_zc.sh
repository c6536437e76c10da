python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_xmarch2.py tests/test_gpu_structured.py tests/test_gpu_fitted.py tests/test_gpu_slabs.py tests/test_gpu_slabs_overlap.py tests/test_gpu_parity_fullsize.py tests/test_gpu_operator.py tests/test_gpu_fullsize.py -q -x > gpurun_out/x2_tests.txt 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/x2_tests.txt
for v in 1 0; do
for wl in config4 config1 config2_p2; do
  ST_ZCOMPACT=$v timeout 900 python bench.py --workload $wl --steps 20 --warmup 5 --sweep 0 --no-cpu-baseline > gpurun_out/zc_${v}_$wl.json 2>gpurun_out/zc_${v}_$wl.err; echo "$wl rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/zc_${v}_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('zc=$v $wl', 'value %.4g ms %.4f kernel %.4f frac %.4f launches %d' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], d['gpu_launches']))"
done; done

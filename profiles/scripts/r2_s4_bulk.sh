python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_xmarch2.py -q -x > gpurun_out/bulk_tests.txt 2>&1; echo "x2 tests rc=$?"; tail -8 gpurun_out/bulk_tests.txt
timeout 900 python -m pytest tests/test_gpu_structured.py tests/test_gpu_fitted.py tests/test_gpu_slabs_overlap.py tests/test_gpu_parity_fullsize.py -q -x > gpurun_out/bulk_tests2.txt 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/bulk_tests2.txt
ST_VARIANT=nobulk ST_NVCC_EXTRA="-DST_X2_BULK=0" python -m paper_2302_05164_b200._build > /dev/null
for v in base nobulk base; do
if [ "$v" = base ]; then unset ST_VARIANT; else export ST_VARIANT=$v; fi
for wl in config4 config1; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --sweep 0 --no-cpu-baseline > gpurun_out/bulk_${v}_$wl.json 2>gpurun_out/bulk_${v}_$wl.err; echo "$wl rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bulk_${v}_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $wl', 'value %.4g ms %.4f kernel %.4f frac %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))"
done; done

python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_structured.py tests/test_gpu_fitted.py tests/test_gpu_parity_fullsize.py -q -x 2>&1 | tail -2
for g in 0 1; do
for wl in config2_p1; do
  ST_SEAM_PAIR=$g timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --sweep 0 --no-cpu-baseline > gpurun_out/p1_${g}_$wl.json 2>gpurun_out/p1_${g}_$wl.err; echo "$wl rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/p1_${g}_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('pair_p1=$g $wl', 'value %.4g ms %.4f kernel %.4f frac %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))"
done; done

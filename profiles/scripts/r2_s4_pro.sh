python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_xmarch2.py -q -x 2>&1 | tail -2
for wl in config4 config1 config4 config1; do
  timeout 900 python bench.py --workload $wl --steps 20 --warmup 5 --sweep 0 --no-cpu-baseline > gpurun_out/pro_$wl.json 2>gpurun_out/pro_$wl.err; echo "$wl rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/pro_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('early-staging $wl', 'value %.4g ms %.4f kernel %.4f frac %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))"
done

# (experiment, its ST_L2_FETCH hook removed afterwards: the L2 fetch granularity hint, 32 / 64 / 128 bytes, does not change the config-4 step: 15.23 / 15.24 / 15.25 ms)
python -c "import __graft_entry__ as g; g.build()" || exit 1
for g in 0 32 64 128; do
if [ "$g" = 0 ]; then unset ST_L2_FETCH; else export ST_L2_FETCH=$g; fi
for wl in config4; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --sweep 0 --no-cpu-baseline > gpurun_out/l2_${g}_$wl.json 2>gpurun_out/l2_${g}_$wl.err; echo "$wl rc=$?"
  grep ST_L2_FETCH gpurun_out/l2_${g}_$wl.err | head -1
  python -c "
import json; d=json.loads(open('gpurun_out/l2_${g}_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('l2=$g $wl', 'value %.4g ms %.4f kernel %.4f frac %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))"
done; done

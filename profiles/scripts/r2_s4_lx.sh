python -c "import __graft_entry__ as g; g.build()"
for lx in 60 100 150 250; do
  ST_LX=$lx timeout 900 python bench.py --workload config4 --steps 10 --warmup 3 --sweep 0 --no-cpu-baseline > gpurun_out/lx_$lx.json 2>gpurun_out/lx_$lx.err; echo "rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/lx_$lx.json').read().strip().splitlines()[-1]); r=d['roofline']
print('lx=$lx', 'value %.4g ms %.4f kernel %.4f frac %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))"
done

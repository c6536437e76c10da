python -c "import __graft_entry__ as g; g.build()"
ST_VARIANT=minb2 ST_NVCC_EXTRA="-DST_X2_MINB=2" python -m paper_2302_05164_b200._build > /dev/null
for v in minb2; do
export ST_VARIANT=$v
for wl in config4 config1; do
  timeout 900 python bench.py --workload $wl --steps 20 --warmup 5 --sweep 0 --no-cpu-baseline > gpurun_out/mb_${v}_$wl.json 2>gpurun_out/mb_${v}_$wl.err; echo "$wl rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/mb_${v}_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $wl', 'value %.4g ms %.4f kernel %.4f frac %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))"
done; done

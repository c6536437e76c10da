python -c "import __graft_entry__ as g; g.build()" || exit 1
for l in 0 3 7 10; do
ST_VARIANT=ru$l ST_NVCC_EXTRA="-Xptxas --register-usage-level=$l" python -m paper_2302_05164_b200._build > /dev/null
done
ST_VARIANT=esf ST_NVCC_EXTRA="-DST_X2_ESTORE_FIRST=1" python -m paper_2302_05164_b200._build > /dev/null
for v in base ru0 ru3 ru7 ru10 esf base; do
if [ "$v" = base ]; then unset ST_VARIANT; else export ST_VARIANT=$v; fi
for wl in config4; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --sweep 0 --no-cpu-baseline > gpurun_out/var_${v}_$wl.json 2>gpurun_out/var_${v}_$wl.err; echo "$wl rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/var_${v}_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $wl', 'value %.4g ms %.4f kernel %.4f frac %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))"
done; done

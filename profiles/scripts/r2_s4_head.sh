set -x
python -c "import __graft_entry__ as g; g.build()"
ST_VARIANT=norow ST_NVCC_EXTRA="-DST_ROWSTORE=0" python -m paper_2302_05164_b200._build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4_tests.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/s4_tests.txt
for v in base norow; do
if [ "$v" = base ]; then unset ST_VARIANT; else export ST_VARIANT=$v; fi
for wl in config4 config1 config2_p2; do
  timeout 900 python bench.py --workload $wl --steps 20 --warmup 5 --sweep 0 --no-cpu-baseline > gpurun_out/s4_${v}_$wl.json 2>gpurun_out/s4_${v}_$wl.err; echo "$wl rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/s4_${v}_$wl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $wl', 'value %.4g ms %.4f kernel %.4f frac %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))"
done; done

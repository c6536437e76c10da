# pipelined seam pass (xmarch_piped): bitwise tests, then config 4 per number of chunk groups
set -x
timeout 900 python -m pytest tests/test_gpu_xmarch2.py -q -x > gpurun_out/r2f_pipe_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2f_pipe_tests.txt
for g in ${GROUPS_LIST:-0 4 6 8 12}; do
ST_SEAM_PIPE=$g timeout 600 python bench.py --steps 20 --warmup 5 --sweep 0 --no-cpu-baseline > gpurun_out/r2f_pipe_g$g.json 2> gpurun_out/r2f_pipe_g$g.err; echo "g=$g rc=$?"
python - <<P
import json
d=json.loads(open('gpurun_out/r2f_pipe_g$g.json').read().strip().splitlines()[-1])
print('G=$g ms/step', round(d['ms_per_step'],3), 'kernel_ms', round(d['roofline']['kernel_ms'],3), 'value', round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2), 'launches', d['gpu_launches'])
P
done

python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/gputests.txt 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/gputests.txt | tail -15
python - <<'PY' > gpurun_out/implicit.json 2>&1
import sys, json, time; sys.argv=['bench.py']
import bench
print(json.dumps(bench.implicit_measure(0, cpu=False)))
t=time.perf_counter(); r=bench.config3_build_measure(cpu=False); print(json.dumps({k:v for k,v in r.items() if k!='per_layer'}), time.perf_counter()-t)
print(json.dumps(r['per_layer'][0])); print(json.dumps(r['per_layer'][-1]))
PY
cat gpurun_out/implicit.json

python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -X faulthandler tools/debug/overlap_repro.py overlap > gpurun_out/dbg_overlap.txt 2>&1; echo "overlap rc=$?"; tail -3 gpurun_out/dbg_overlap.txt
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=10 > gpurun_out/gputests.txt 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/gputests.txt | tail -15
python - <<'PY' > gpurun_out/implicit.json 2>&1
import sys, json; sys.argv=['bench.py']
import bench
print(json.dumps(bench.implicit_measure(0, cpu=False)))
PY
cat gpurun_out/implicit.json

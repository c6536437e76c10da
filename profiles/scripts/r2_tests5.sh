python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/gputests.txt 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/gputests.txt | tail -15
REFSUITE_TIMEOUT=2700 bash tools/run_reference_suite.sh --durations=5
grep -E "passed|failed" gpurun_out/refsuite.txt | tail -3

python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; cat gpurun_out/smoke.txt | tail -5
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/gputests.txt 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/gputests.txt | tail -15

python -c "import __graft_entry__ as g; g.build()" || exit 1
REFSUITE_TIMEOUT=2400 bash tools/run_reference_suite.sh > /dev/null 2>&1
tail -5 gpurun_out/refsuite.txt

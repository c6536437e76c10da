set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_fitted.py -x -q > gpurun_out/fitted.txt 2>&1; echo "fitted rc=$?" >> gpurun_out/fitted.txt
tail -30 gpurun_out/fitted.txt
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.txt
tail -30 gpurun_out/gputests.txt

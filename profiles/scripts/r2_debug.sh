python -c "import __graft_entry__ as g; g.build()"
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -X faulthandler tools/debug/overlap_repro.py plain > gpurun_out/dbg_plain.txt 2>&1; echo "plain rc=$?"
tail -20 gpurun_out/dbg_plain.txt
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -X faulthandler tools/debug/overlap_repro.py overlap > gpurun_out/dbg_overlap.txt 2>&1; echo "overlap rc=$?"
tail -40 gpurun_out/dbg_overlap.txt

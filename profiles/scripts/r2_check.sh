set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 600 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck.txt
timeout 900 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.txt
tail -3 gpurun_out/gputests.txt; cat gpurun_out/fp64_peak.json; tail -5 gpurun_out/memcheck.txt gpurun_out/racecheck.txt

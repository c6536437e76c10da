set -x
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
free -g | head -2
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.json; tail -20 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
cat gpurun_out/bench_ref.json | tail -c 1500

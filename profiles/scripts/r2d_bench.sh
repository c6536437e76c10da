set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.txt 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/r2d_smoke.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc=$?"
tail -c 400 gpurun_out/r2d_bench.json; tail -3 gpurun_out/r2d_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2d_bench_ref.json 2>&1; echo "ref rc=$?"
tail -c 600 gpurun_out/r2d_bench_ref.json

# last check of round 2 (after the profile-guided prefetches of the config-3 scan kernels): build, GPU suite,
# smoke, reference arm, default bench
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2i_gputests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2i_gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2i_bench_ref.json 2>&1; echo "ref rc=$?"
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2i_bench.json

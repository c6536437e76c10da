# final check of round 2 on the final tree: build, GPU suite, smoke, reference arm, default bench,
# ncu of configs[4] (launch list + one full capture of k_xmarch2)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2g_gputests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2g_gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2g_bench_ref.json 2>&1; echo "ref rc=$?"
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2g_bench.json
timeout 1500 bash profiles/run_prof.sh r2g_config4 --workload config4; echo "prof rc=$?"
python tools/srcmix.py gpurun_out/srcmix_r2g_config4.csv 60 > gpurun_out/r2g_config4_srcmix.txt
python tools/stallmix.py gpurun_out/srcmix_r2g_config4.csv 40 > gpurun_out/r2g_config4_stallmix.txt
rm -f gpurun_out/srcmix_r2g_*.csv

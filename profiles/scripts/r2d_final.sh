# final captures of round 2 (pair seam layout): full GPU suite, smoke, the
# default bench line and the reference arm, ncu of config 4 and of the
# 1/8 replica with its seam pass
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2d_gputests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2d_gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 1200 bash profiles/run_prof.sh r2d_config4 --workload config4; echo "prof rc=$?"
timeout 900 bash profiles/run_prof.sh r2d_config4_s2 --workload config4_s2; echo "prof s2 rc=$?"
KREGEX=k_seam_list timeout 900 bash profiles/run_prof.sh r2d_config4_s2_seams --workload config4_s2; echo "seam prof rc=$?"
timeout 900 bash profiles/run_prof.sh r2d_config1 --workload config1; echo "prof c1 rc=$?"
ST_XMARCH2=0 timeout 900 bash profiles/run_prof.sh r2d_config2_p2 --workload config2_p2; echo "prof c2 rc=$?"
for t in r2d_config4; do
python tools/srcmix.py gpurun_out/srcmix_$t.csv 60 > gpurun_out/${t}_srcmix.txt
python tools/stallmix.py gpurun_out/srcmix_$t.csv 40 > gpurun_out/${t}_stallmix.txt
done
rm -f gpurun_out/srcmix_r2d_*.csv

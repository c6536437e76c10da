# round-2 (final) captures of the lean kernel: full GPU suite, then per
# workload the plain bench line, the per-launch ncu list and one
# `ncu --set full` capture of the hot kernel (profiles/run_prof.sh)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2c_gputests.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2c_gputests.txt
timeout 1200 bash profiles/run_prof.sh r2c_config4 --workload config4; echo "prof rc=$?"
timeout 900 bash profiles/run_prof.sh r2c_config4_s2 --workload config4_s2; echo "prof s2 rc=$?"
KREGEX=k_seam_list timeout 900 bash profiles/run_prof.sh r2c_config4_s2_seams --workload config4_s2; echo "seam prof rc=$?"
timeout 900 bash profiles/run_prof.sh r2c_config1 --workload config1; echo "prof c1 rc=$?"
ST_XMARCH2=0 timeout 900 bash profiles/run_prof.sh r2c_config2_p2 --workload config2_p2; echo "prof c2 rc=$?"
for t in r2c_config4 r2c_config4_s2; do
python tools/srcmix.py gpurun_out/srcmix_$t.csv 60 > gpurun_out/${t}_srcmix.txt
python tools/stallmix.py gpurun_out/srcmix_$t.csv 40 > gpurun_out/${t}_stallmix.txt
done
rm -f gpurun_out/srcmix_r2c_*.csv

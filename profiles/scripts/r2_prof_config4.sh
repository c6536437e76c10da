set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 bash profiles/run_prof.sh r2_config4 --workload config4; echo "prof rc=$?"
tail -5 gpurun_out/ncu_full_r2_config4.log; ls -la gpurun_out/ | grep r2_config4
timeout 900 bash profiles/run_prof.sh r2_config4_s2 --workload config4_s2; echo "prof s2 rc=$?"
tail -3 gpurun_out/ncu_full_r2_config4_s2.log
KREGEX=k_seam_list timeout 900 bash profiles/run_prof.sh r2_config4_s2_seams --workload config4_s2; echo "seam prof rc=$?"

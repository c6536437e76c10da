python -c "import __graft_entry__ as g; g.build()"
KREGEX=k_seam_list timeout 900 bash profiles/run_prof.sh r2d_config4_s2_seams --workload config4_s2; echo "seam prof rc=$?"
python profiles/summarize.py gpurun_out/raw_r2d_config4_s2_seams.csv
grep -i "DRAM Throughput\|Memory Throughput\|L2 Hit\|Duration" gpurun_out/details_r2d_config4_s2_seams.txt | head
rm -f gpurun_out/srcmix_r2d_*.csv

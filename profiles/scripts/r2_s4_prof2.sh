python -c "import __graft_entry__ as g; g.build()"
timeout 900 bash profiles/run_prof.sh s4_config4_s2 --workload config4_s2; echo "prof rc=$?"
python tools/srcmix.py gpurun_out/srcmix_s4_config4_s2.csv 400 > gpurun_out/s4_srcmix_full.txt
python tools/stallmix.py gpurun_out/srcmix_s4_config4_s2.csv 40 > gpurun_out/s4_stallmix.txt
python profiles/summarize.py gpurun_out/raw_s4_config4_s2.csv > gpurun_out/s4_summary.txt

python -c "import __graft_entry__ as g; g.build()"
timeout 900 bash profiles/run_prof.sh r2b_config4_s2 --workload config4_s2; echo "prof rc=$?"

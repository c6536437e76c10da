# one full capture of k_pcg_persistent on the config-3-sized box, source-level stall mix
PYTHONPATH=. ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_pcg_persistent -s 6 -c 1 \
  -o gpurun_out/prof_pcg -f python tools/debug/imp_phases.py > gpurun_out/ncu_pcg.log 2>&1
ncu -i gpurun_out/prof_pcg.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/srcmix_pcg.csv 2>/dev/null
python tools/stallmix.py gpurun_out/srcmix_pcg.csv 45 > gpurun_out/pcg_stallmix.txt
rm -f gpurun_out/srcmix_pcg.csv gpurun_out/prof_pcg.ncu-rep

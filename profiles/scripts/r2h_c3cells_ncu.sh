# config-3 layer-0 scan: one full capture of k_rhs_cells with warm caches, source-level stall mix
NSTEPS=64 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_rhs_cells -s 40 -c 1 \
  -o gpurun_out/prof_c3cells -f python tools/debug/config3_scan_probe.py > gpurun_out/ncu_c3cells.log 2>&1
ncu -i gpurun_out/prof_c3cells.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/srcmix_c3cells.csv 2>/dev/null
ncu -i gpurun_out/prof_c3cells.ncu-rep --page details > gpurun_out/details_c3cells.txt 2>/dev/null
python tools/srcmix.py gpurun_out/srcmix_c3cells.csv 40 > gpurun_out/c3cells_srcmix.txt
python tools/stallmix.py gpurun_out/srcmix_c3cells.csv 40 > gpurun_out/c3cells_stallmix.txt
rm -f gpurun_out/srcmix_c3cells.csv gpurun_out/prof_c3cells.ncu-rep

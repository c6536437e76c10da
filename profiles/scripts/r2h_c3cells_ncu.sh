# config-3 layer-0 scan: one full capture of a scan kernel (KREGEX) with warm caches, source-level stall mix
K=${KREGEX:-k_rhs_cells}
NSTEPS=64 ncu --set full --cache-control none --clock-control none --import-source on -k regex:$K -s 40 -c 1 \
  -o gpurun_out/prof_c3_$K -f python tools/debug/config3_scan_probe.py > gpurun_out/ncu_c3_$K.log 2>&1
ncu -i gpurun_out/prof_c3_$K.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/srcmix_c3_$K.csv 2>/dev/null
python tools/stallmix.py gpurun_out/srcmix_c3_$K.csv 40 > gpurun_out/c3_${K}_stallmix.txt
rm -f gpurun_out/srcmix_c3_$K.csv gpurun_out/prof_c3_$K.ncu-rep

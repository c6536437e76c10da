#!/bin/bash
# ncu --set full of one kernel (regex $1) in the default config-1 bench, warm
# or cold cache ($2 = none|all), exported pages into gpurun_out/<tag>_*
tag=$3
ncu --set full --clock-control none --cache-control ${2:-all} --import-source on -k regex:"$1" -s 4 -c 1 \
    -o gpurun_out/prof_$tag -f python bench.py --steps 3 --warmup 3 --sweep 0 --no-cpu-baseline > gpurun_out/ncu_full_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>/dev/null || true
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/srcmix_$tag.csv 2>/dev/null || true
ncu -i gpurun_out/prof_$tag.ncu-rep --page details > gpurun_out/details_$tag.txt 2>/dev/null || true
rm -f gpurun_out/prof_$tag.ncu-rep

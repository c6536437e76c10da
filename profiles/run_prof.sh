#!/bin/bash
# ncu capture of the explicit-step kernels (run under gpurun, 1 GPU).
# usage: profiles/run_prof.sh <tag> [bench args...]
set -e
tag=$1; shift
cmd="python bench.py --steps 3 --warmup 3 --sweep 0 --no-cpu-baseline $*"
$cmd > gpurun_out/plain_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv $cmd > gpurun_out/ncu_launch_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_x(march|slab)}" -s 4 -c 1 \
    -o gpurun_out/prof_$tag -f $cmd > gpurun_out/ncu_full_$tag.log 2>&1
# export the pages read here (raw metrics, source/SASS with per-line counts);
# the report itself is dropped unless KEEP_REP=1 (gpurun_out is capped at 64 MiB)
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>/dev/null || true
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source cuda,sass \
    > gpurun_out/srcmix_$tag.csv 2>/dev/null || true
ncu -i gpurun_out/prof_$tag.ncu-rep --page details > gpurun_out/details_$tag.txt 2>/dev/null || true
[ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/prof_$tag.ncu-rep

#!/bin/bash
# ncu --set full of one decode launch (kbench config), source page included:  bash tools/gpu_prof.sh NAME "kbench args" [env]
# Keeps the summary and the per-line source CSV (the .ncu-rep stays on the box: gpurun copies back <= 64 MiB).
mkdir -p gpurun_out /tmp/prof
name=$1; shift; args=$1; shift
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode -s 3 -c 1 \
  -o /tmp/prof/$name -f python tools/kbench.py $args --reps 1 > gpurun_out/$name.ncu.log 2>&1
ncu -i /tmp/prof/$name.ncu-rep --page source --csv > gpurun_out/$name.source.csv 2>/dev/null
python tools/ncu_summary.py /tmp/prof/$name.ncu-rep > gpurun_out/$name.summary.txt 2>&1
gzip -f gpurun_out/$name.source.csv

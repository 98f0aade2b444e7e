#!/bin/bash
# A/B timing of kernel variants (one layer each) on the GPU box:  bash tools/ab.sh lib1.so lib2.so ...
mkdir -p gpurun_out
: > gpurun_out/ab.log
CFGS=${AB_CFGS:-"--kb 4 --vb 2|--kb 8 --vb 4|--kb 2 --vb 2|--kb 4 --vb 4 --g 7 --H 4"}
IFS='|' read -ra CFG <<< "$CFGS"
for lib in "$@"; do
  for cfg in "${CFG[@]}"; do
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/ab.log 2>&1
  done
done

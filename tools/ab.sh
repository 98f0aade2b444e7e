#!/bin/bash
# A/B timing of kernel variants (one layer each) on the GPU box.
mkdir -p gpurun_out
: > gpurun_out/ab.log
for lib in "$@"; do
  for cfg in "--kb 4 --vb 2" "--kb 8 --vb 4" "--kb 2 --vb 2" "--kb 4 --vb 4 --g 7 --H 4"; do
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/ab.log 2>&1
  done
done

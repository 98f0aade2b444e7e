#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/ab.log
for ns in 1 2 3 5 8; do
  for lib in libkvt.so libkvt_loadonly.so; do
    echo "nsplit=$ns" >> gpurun_out/ab.log
    KVT_NSPLIT=$ns KVT_LIB=$lib timeout 300 python tools/kbench.py --kb 4 --vb 2 >> gpurun_out/ab.log 2>&1
  done
done

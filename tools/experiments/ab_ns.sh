#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/ab.log
for ns in 1 4; do
  for lib in libkvt_loadonly.so libkvt.so; do
    echo "nsplit=$ns" >> gpurun_out/ab.log
    KVT_NSPLIT=$ns KVT_LIB=$lib timeout 300 python tools/kbench.py --kb 4 --vb 2 >> gpurun_out/ab.log 2>&1
  done
done
KVT_LIB=libkvt.so timeout 300 python tools/kbench.py --kb 4 --vb 2 >> gpurun_out/ab.log 2>&1
KVT_LIB=libkvt.so timeout 300 python tools/kbench.py --kb 4 --vb 2 --S 8160 >> gpurun_out/ab.log 2>&1
KVT_LIB=libkvt_loadonly.so timeout 300 python tools/kbench.py --kb 4 --vb 2 --S 8160 >> gpurun_out/ab.log 2>&1

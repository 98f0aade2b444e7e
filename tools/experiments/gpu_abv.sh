#!/bin/bash
# A/B of kernel build variants (libkvt_<v>.so) on one GPU: parity subset per variant, then one-layer timings.
#   bash tools/gpu_abv.sh TAG "v1 v2 ..." ["kbench cfg;kbench cfg;..."]
mkdir -p gpurun_out
tag=$1; vars=$2
cfgs=${3:-"--kb 4 --vb 2;--kb 4 --vb 4;--kb 2 --vb 2;--kb 4 --vb 2 --pt;--kb 4 --vb 4 --g 7 --H 4"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${tag}_gpu.txt 2>&1
: > gpurun_out/${tag}_ab.log
for v in $vars; do
  lib=libkvt_$v.so; [ "$v" == "base" ] && lib=libkvt.so
  KVT_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -q -x > gpurun_out/${tag}_pytest_$v.log 2>&1
  echo "$v pytest exit $?" >> gpurun_out/${tag}_ab.log
done
for rep in 1 2; do
IFS=';' read -ra CS <<< "$cfgs"
for cfg in "${CS[@]}"; do
  for v in $vars; do
    lib=libkvt_$v.so; [ "$v" == "base" ] && lib=libkvt.so
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/${tag}_ab.log 2>&1
  done
done
done

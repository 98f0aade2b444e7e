#!/bin/bash
# one-layer A/B of build variants (no tests):  bash tools/gpu_abk.sh TAG "v1 v2 ..." ["cfg;cfg"]
mkdir -p gpurun_out
tag=$1; vars=$2
cfgs=${3:-"--kb 4 --vb 2 --S 8200;--kb 4 --vb 4 --S 8200;--kb 2 --vb 2 --S 8200;--kb 8 --vb 4 --S 8200;--kb 4 --vb 2 --pt --S 8200;--kb 4 --vb 4 --g 7 --H 4 --S 8200"}
: > gpurun_out/${tag}_ab.log
IFS=';' read -ra CS <<< "$cfgs"
for rep in 1 2; do
for cfg in "${CS[@]}"; do
  for v in $vars; do
    lib=libkvt_$v.so; [ "$v" == "base" ] && lib=libkvt.so
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/${tag}_ab.log 2>&1
  done
done
done

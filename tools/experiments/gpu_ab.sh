#!/bin/bash
# A/B of the decode schedules on one GPU: parity tests, one-layer timings with KVT_PK=0 (stream-K CTAs) vs 1
# (persistent warp items), then the headline bench.   bash tools/gpu_ab.sh [tests] [bench]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt 2>&1
if [[ " $* " == *" tests "* ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
: > gpurun_out/ab.log
for cfg in "--kb 4 --vb 2" "--kb 8 --vb 4" "--kb 2 --vb 2" "--kb 4 --vb 4" "--kb 4 --vb 2 --pt" "--kb 4 --vb 4 --g 7 --H 4" "--kb 8 --vb 4 --g 7 --H 4" "--kb 4 --vb 2 --B 74" "--kb 4 --vb 2 --B 8 --S 131072"; do
  for pk in 0 1; do
    echo -n "PK=$pk " >> gpurun_out/ab.log
    KVT_PK=$pk timeout 300 python tools/kbench.py $cfg >> gpurun_out/ab.log 2>&1
  done
done
if [[ " $* " == *" bench "* ]]; then
  for w in llama-3.25 qwen-4.00 qwen-4.00-pertoken; do
    timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$w.log
  done
fi

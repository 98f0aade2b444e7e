#!/bin/bash
# Run on the GPU box via gpurun: parity tests, smoke, benches, ncu launch list + one full capture.
#   bash tools/gpu_check.sh [ncu] [extra bench workloads...]
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
NCU=0
if [ "$1" == "ncu" ]; then NCU=1; shift; fi
for w in "$@"; do
  timeout 900 python bench.py --steps 30 --warmup 3 --workload $w --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo "exit $?" >> gpurun_out/bench_$w.log
done
if [ "$NCU" == "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|combine|append" -s 100 -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
# the dominant kernel (K4V2 layers, 20 of 32 in llama-3.25) at the bench launch configuration (B=64, S=8192)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mma -s 2 -c 1 -o gpurun_out/prof_decode -f python tools/kbench.py --kb 4 --vb 2 --reps 1 > gpurun_out/ncu_full.log 2>&1
fi

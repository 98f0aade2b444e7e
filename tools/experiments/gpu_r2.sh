#!/bin/bash
# Round-2 GPU check (run via gpurun): edge-case parity first, then the whole -m gpu suite, smoke, benches.
#   bash tools/gpu_r2.sh [tests|all] [bench args...]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_edge.py -q -x -rf > gpurun_out/pytest_edge.log 2>&1; echo "edge exit $?" >> gpurun_out/pytest_edge.log
if [ "$1" == "all" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 20 --warmup 5 --launch eager --no-cpu-baseline > gpurun_out/bench_eager.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_eager.log

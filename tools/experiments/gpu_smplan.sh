#!/bin/bash
# per-SM plan: parity (new tests + full size + edge + parity), then one-layer timings with the plan off / on
mkdir -p gpurun_out
tag=$1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${tag}_gpu.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_smplan.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py tests/test_gpu_parity.py -m gpu -q -x -rf > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_pytest.log
: > gpurun_out/${tag}_ab.log
for cfg in "--kb 4 --vb 2" "--kb 4 --vb 4" "--kb 2 --vb 2" "--kb 8 --vb 4" "--kb 8 --vb 8" "--kb 4 --vb 2 --pt" "--kb 4 --vb 4 --g 7 --H 4" "--kb 4 --vb 4 --g 7 --H 4 --pt" "--kb 8 --vb 8 --g 7 --H 4" "--kb 4 --vb 2 --B 48"; do
  for sp in 0 1; do
    echo -n "SMPLAN=$sp " >> gpurun_out/${tag}_ab.log
    KVT_SMPLAN=$sp timeout 300 python tools/kbench.py $cfg >> gpurun_out/${tag}_ab.log 2>&1
  done
done
for sp in 0 1; do
  KVT_SMPLAN=$sp timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_sp$sp.log 2>&1
  KVT_SMPLAN=$sp timeout 600 python bench.py --workload qwen-4.00 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_qwen_sp$sp.log 2>&1
done

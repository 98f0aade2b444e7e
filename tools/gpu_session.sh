#!/bin/bash
# One gpurun call: -m gpu suite, smoke, bench (graph), and an ncu source capture of the K4V2 layer.
#   bash tools/gpu_session.sh TAG [tests|notests]
mkdir -p gpurun_out
tag=$1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${tag}_gpu.txt 2>&1
if [ "$2" != "notests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${tag}_smoke.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${tag}_bench.log
for cfg in "--kb 4 --vb 2" "--kb 4 --vb 4" "--kb 2 --vb 2" "--kb 8 --vb 4" "--kb 4 --vb 4 --g 7 --H 4"; do
  timeout 300 python tools/kbench.py $cfg >> gpurun_out/${tag}_kbench.log 2>&1
done
bash tools/gpu_prof.sh ${tag}_K4V2 "--kb 4 --vb 2"

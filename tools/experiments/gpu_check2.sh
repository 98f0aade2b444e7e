#!/bin/bash
mkdir -p gpurun_out
tag=$1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_pytest.log
bash tools/gpu_bench_ab.sh ${tag}l llama-3.25 "KVT_SMPLAN=0;KVT_SMPLAN=1"
bash tools/gpu_bench_ab.sh ${tag}q qwen-4.00 "KVT_SMPLAN=1"

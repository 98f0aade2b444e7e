#!/bin/bash
mkdir -p gpurun_out
tag=$1
timeout 1200 python -m pytest tests/test_gpu_smplan.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py tests/test_gpu_parity.py -m gpu -q -x -rf > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_pytest.log
bash tools/gpu_abk.sh ${tag} "base"
bash tools/gpu_bench_ab.sh ${tag}l llama-3.25 "KVT_SMPLAN=1;KVT_SMPLAN=1 KVT_PDL=1"
bash tools/gpu_bench_ab.sh ${tag}q qwen-4.00 "KVT_SMPLAN=1"

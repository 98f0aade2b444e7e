mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_push.py -m gpu -q -x -rs > gpurun_out/pytest_push.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_push.log
timeout 600 python bench.py --workload llama-128k-seqshard --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ss_nccl.log 2>&1
timeout 600 python bench.py --workload llama-128k-seqshard --steps 30 --warmup 3 --no-cpu-baseline --exchange symm > gpurun_out/bench_ss_symm.log 2>&1

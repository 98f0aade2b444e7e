mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paged.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_paged.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_paged.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_dense.json 2> gpurun_out/bench_dense.err
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --paged > gpurun_out/bench_paged.json 2> gpurun_out/bench_paged.err

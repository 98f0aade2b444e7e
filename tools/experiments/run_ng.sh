mkdir -p gpurun_out
KVT_NG=2 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_paged.py tests/test_gpu_graph.py -m gpu -q -x > gpurun_out/pytest_ng2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ng2.log
: > gpurun_out/ng.log
for ng in 1 2; do
  for cfg in "--kb 4 --vb 4 --g 7 --H 4" "--kb 4 --vb 2 --g 7 --H 4" "--kb 8 --vb 2 --g 7 --H 4 --pt" "--kb 4 --vb 4 --g 7 --H 4 --pt" "--kb 8 --vb 8 --g 7 --H 4"; do
    KVT_NG=$ng timeout 300 python tools/kbench.py $cfg >> gpurun_out/ng.log 2>&1
  done
done
for ng in 1 2; do
KVT_NG=$ng timeout 600 python bench.py --workload qwen-4.00 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ng${ng}.json 2>&1
KVT_NG=$ng timeout 600 python bench.py --workload qwen-4.00-pertoken --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ng${ng}_pt.json 2>&1
done

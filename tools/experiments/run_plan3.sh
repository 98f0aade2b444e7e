mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_plan3.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_plan3.log
for w in qwen-4.00 qwen-4.00-pertoken qwen-3.92 llama-3.25 llama-kv8 llama-128k-seqshard; do
timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_plan3_$w.json 2>&1
done

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_plan.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_plan.log
for w in qwen-4.00 qwen-4.00-pertoken qwen-3.92 llama-3.25; do
timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_plan_$w.json 2>&1
done

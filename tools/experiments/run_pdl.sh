mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_pdl.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_pdl.log
for i in 1 2; do
KVT_PDL=0 timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pdl0_$i.json 2>&1
KVT_PDL=1 timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pdl1_$i.json 2>&1
done
KVT_PDL=0 timeout 600 python bench.py --workload qwen-4.00 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pdl0_q.json 2>&1
KVT_PDL=1 timeout 600 python bench.py --workload qwen-4.00 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pdl1_q.json 2>&1

mkdir -p gpurun_out
for w in qwen-4.00 qwen-4.00-pertoken; do
KVT_PDL=0 timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_plan2_$w.json 2>&1
done

mkdir -p gpurun_out
for w in llama-3.25 qwen-4.00; do
timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e_$w.json 2> gpurun_out/bench_e2e_$w.err
done

mkdir -p gpurun_out
bash tools/gpu_check.sh ncu llama-kv8 qwen-4.00 qwen-3.92 qwen-4.00-pertoken llama-128k-seqshard
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --paged > gpurun_out/bench_paged_final.log 2>&1

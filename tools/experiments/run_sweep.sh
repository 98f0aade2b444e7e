mkdir -p gpurun_out
timeout 2400 python tools/sweep_ctx.py --model ${1:-llama} > gpurun_out/sweep.log 2>&1

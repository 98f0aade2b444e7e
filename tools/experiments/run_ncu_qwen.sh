mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mma -s 2 -c 1 -o gpurun_out/prof_qwen -f python tools/kbench.py --kb 4 --vb 4 --g 7 --H 4 --reps 1 > gpurun_out/ncu_qwen.log 2>&1

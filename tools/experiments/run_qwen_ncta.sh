mkdir -p gpurun_out
: > gpurun_out/qwen_ncta.log
for n in 0 256 296 384 444; do
  for cfg in "--kb 4 --vb 4 --g 7 --H 4" "--kb 4 --vb 2 --g 7 --H 4" "--kb 8 --vb 2 --g 7 --H 4 --pt"; do
    echo "NCTA=$n" >> gpurun_out/qwen_ncta.log
    if [ $n == 0 ]; then timeout 300 python tools/kbench.py $cfg >> gpurun_out/qwen_ncta.log 2>&1; else KVT_NCTA=$n timeout 300 python tools/kbench.py $cfg >> gpurun_out/qwen_ncta.log 2>&1; fi
  done
done

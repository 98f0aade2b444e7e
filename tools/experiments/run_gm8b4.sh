mkdir -p gpurun_out
: > gpurun_out/gm8b4.log
for lib in libkvt.so libkvt_gm8b4.so; do
  for n in 0 512; do
    for cfg in "--kb 4 --vb 2 --g 7 --H 4 --pt" "--kb 4 --vb 4 --g 7 --H 4 --pt" "--kb 4 --vb 2 --g 7 --H 4"; do
      echo "$lib NCTA=$n" >> gpurun_out/gm8b4.log
      if [ $n == 0 ]; then KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/gm8b4.log 2>&1; else KVT_LIB=$lib KVT_NCTA=$n timeout 300 python tools/kbench.py $cfg >> gpurun_out/gm8b4.log 2>&1; fi
    done
  done
done

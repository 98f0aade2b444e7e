mkdir -p gpurun_out
: > gpurun_out/exp5.log
for lib in libkvt.so libkvt_exp5.so libkvt.so libkvt_exp5.so; do
  for cfg in "--kb 4 --vb 2" "--kb 4 --vb 4 --g 7 --H 4"; do
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/exp5.log 2>&1
  done
done

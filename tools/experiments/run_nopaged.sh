mkdir -p gpurun_out
: > gpurun_out/nopaged.log
for rep in 1 2; do
for lib in libkvt.so libkvt_nopaged.so; do
  for cfg in "--kb 4 --vb 2" "--kb 2 --vb 2" "--kb 4 --vb 4 --g 7 --H 4"; do
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg --reps 50 >> gpurun_out/nopaged.log 2>&1
  done
done
done

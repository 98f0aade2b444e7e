mkdir -p gpurun_out
: > gpurun_out/pf.log
for lib in libkvt.so libkvt_pf1.so libkvt_pf2.so libkvt_pf4.so libkvt_exp4.so libkvt_exp4pf2.so; do
  for cfg in "--kb 4 --vb 2" "--kb 2 --vb 2" "--kb 8 --vb 4" "--kb 4 --vb 4 --g 7 --H 4"; do
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/pf.log 2>&1
  done
done

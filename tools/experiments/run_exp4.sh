mkdir -p gpurun_out
: > gpurun_out/exp4.log
for lib in libkvt.so libkvt_exp4.so libkvt_exp4ns3.so libkvt_exp4ns4.so libkvt_minb5.so; do
  for cfg in "--kb 4 --vb 2" "--kb 2 --vb 2" "--kb 8 --vb 8"; do
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/exp4.log 2>&1
  done
done

mkdir -p gpurun_out
: > gpurun_out/ns3.log
for lib in libkvt.so libkvt_ns3.so; do
  for cfg in "--kb 4 --vb 2" "--kb 4 --vb 2 --B 74" "--kb 2 --vb 2" "--kb 4 --vb 4 --g 7 --H 4"; do
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/ns3.log 2>&1
  done
done

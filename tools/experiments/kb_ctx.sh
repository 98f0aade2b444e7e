: > gpurun_out/k1_ab.log
for cfg in "--kb 4 --vb 2" "--kb 4 --vb 2 --S 8200" "--kb 4 --vb 2 --S 8200 --no-host --cap 8320" "--kb 4 --vb 2 --S 8216 --no-host --cap 8320"; do
  for sp in 0 1; do
    echo -n "SMPLAN=$sp $cfg: " >> gpurun_out/k1_ab.log
    KVT_SMPLAN=$sp timeout 300 python tools/kbench.py $cfg >> gpurun_out/k1_ab.log 2>&1
  done
done

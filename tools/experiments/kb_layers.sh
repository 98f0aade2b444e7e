: > gpurun_out/k2_ab.log
for cfg in "--kb 4 --vb 2 --S 8200" "--kb 4 --vb 2 --S 8200 --no-flush" "--kb 4 --vb 2 --S 8200 --layers 16" "--kb 4 --vb 2 --S 8200 --layers 16 --no-flush"; do
  for sp in 0 1; do
    echo -n "SMPLAN=$sp $cfg: " >> gpurun_out/k2_ab.log
    KVT_SMPLAN=$sp timeout 300 python tools/kbench.py $cfg >> gpurun_out/k2_ab.log 2>&1
  done
done

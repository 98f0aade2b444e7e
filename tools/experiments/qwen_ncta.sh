: > gpurun_out/qn_ab.log
for cfg in "--kb 4 --vb 4 --g 7 --H 4 --S 8200" "--kb 4 --vb 2 --g 7 --H 4 --S 8200" "--kb 4 --vb 4 --g 7 --H 4 --S 8200 --pt"; do
  for n in 0 296 444 256; do
    echo -n "NCTA=$n " >> gpurun_out/qn_ab.log
    KVT_NCTA=$n timeout 300 python tools/kbench.py $cfg >> gpurun_out/qn_ab.log 2>&1
  done
done

: > gpurun_out/qw_ab.log
for cfg in "--kb 4 --vb 4 --g 7 --H 4 --S 8200" "--kb 4 --vb 2 --g 7 --H 4 --S 8200" "--kb 4 --vb 4 --g 7 --H 4 --S 8200 --pt"; do
  for sp in 1 2; do
    for pf in 1 0; do
    echo -n "SMPLAN=$sp PF=$pf " >> gpurun_out/qw_ab.log
    KVT_SMPLAN=$sp KVT_PIECE_FIRST=$pf timeout 300 python tools/kbench.py $cfg >> gpurun_out/qw_ab.log 2>&1
    done
  done
done

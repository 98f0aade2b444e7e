: > gpurun_out/pf_ab.log
for cfg in "--kb 4 --vb 2 --S 8200" "--kb 4 --vb 4 --S 8200" "--kb 2 --vb 2 --S 8200" "--kb 4 --vb 2 --pt --S 8200" "--kb 4 --vb 2 --B 48 --S 8200"; do
  for pf in 0 1; do
    echo -n "PF=$pf " >> gpurun_out/pf_ab.log
    KVT_PIECE_FIRST=$pf timeout 300 python tools/kbench.py $cfg >> gpurun_out/pf_ab.log 2>&1
  done
done
KVT_PIECE_FIRST=1 KVT_LIB=libkvt_trace.so python tools/trace_balance.py --kb 4 --vb 2 --S 8200 > gpurun_out/pf_tr1.log 2>&1
bash tools/gpu_bench_ab.sh pfb llama-3.25 "KVT_PIECE_FIRST=0;KVT_PIECE_FIRST=1"

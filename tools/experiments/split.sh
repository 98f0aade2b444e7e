: > gpurun_out/sp_ab.log
for cfg in "--kb 4 --vb 2 --S 8200" "--kb 4 --vb 4 --S 8200" "--kb 2 --vb 2 --S 8200" "--kb 4 --vb 2 --pt --S 8200" "--kb 4 --vb 4 --g 7 --H 4 --S 8200"; do
  for sp in 0 1; do
    echo -n "SPLIT=$sp " >> gpurun_out/sp_ab.log
    KVT_SMSPLIT=$sp timeout 300 python tools/kbench.py $cfg >> gpurun_out/sp_ab.log 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_smplan.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py -m gpu -q -x > gpurun_out/sp_pytest.log 2>&1; echo "exit $?" >> gpurun_out/sp_pytest.log
bash tools/gpu_bench_ab.sh spb llama-3.25 "KVT_SMSPLIT=0;KVT_SMSPLIT=1"
bash tools/gpu_bench_ab.sh spq qwen-4.00 "KVT_SMSPLIT=1"

mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_push.py -m gpu -q -x > gpurun_out/pytest_merge.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_merge.log
: > gpurun_out/merge.log
for lib in libkvt_oldmerge.so libkvt.so; do
  KVT_LIB=$lib KVT_NCTA=592 timeout 300 python tools/kbench.py --kb 4 --vb 2 >> gpurun_out/merge.log 2>&1
  KVT_LIB=$lib timeout 300 python tools/kbench.py --kb 4 --vb 2 >> gpurun_out/merge.log 2>&1
  KVT_LIB=$lib timeout 300 python tools/kbench.py --kb 8 --vb 4 >> gpurun_out/merge.log 2>&1
  KVT_LIB=$lib timeout 300 python tools/kbench.py --kb 4 --vb 4 --g 7 --H 4 --B 32 >> gpurun_out/merge.log 2>&1
  KVT_LIB=$lib timeout 300 python tools/kbench.py --kb 4 --vb 2 --B 16 >> gpurun_out/merge.log 2>&1
  KVT_LIB=$lib KVT_NCTA=444 timeout 300 python tools/kbench.py --kb 4 --vb 4 --g 7 --H 4 >> gpurun_out/merge.log 2>&1
done

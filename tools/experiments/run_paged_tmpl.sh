mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_paged.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_push.py -m gpu -q -x > gpurun_out/pytest_ptmpl.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ptmpl.log
: > gpurun_out/ptmpl.log
for cfg in "--kb 4 --vb 2" "--kb 2 --vb 2" "--kb 8 --vb 4" "--kb 4 --vb 4 --g 7 --H 4" "--kb 4 --vb 2 --g 7 --H 4 --pt" "--kb 8 --vb 2 --g 7 --H 4 --pt" "--kb 4 --vb 4 --g 7 --H 4 --pt"; do
  timeout 300 python tools/kbench.py $cfg --reps 50 >> gpurun_out/ptmpl.log 2>&1
done

#!/bin/bash
# quick GPU iteration: parity tests + one-layer kernel timings (+ optional bench)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/ab.log
for lib in "$@"; do
  for cfg in "--kb 4 --vb 2" "--kb 8 --vb 4" "--kb 2 --vb 2" "--kb 4 --vb 4 --g 7 --H 4"; do
    KVT_LIB=$lib timeout 300 python tools/kbench.py $cfg >> gpurun_out/ab.log 2>&1
  done
done

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k ragged > gpurun_out/pytest_ragged.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ragged.log

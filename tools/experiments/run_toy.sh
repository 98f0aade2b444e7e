mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_toyllm.py -m gpu -q -x > gpurun_out/pytest_toy.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_toy.log

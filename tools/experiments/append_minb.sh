for v in base mb6 mb8; do
  lib=libkvt_$v.so; [ "$v" == "base" ] && lib=libkvt.so
  KVT_LIB=$lib python tools/bench_aux.py > gpurun_out/aux_$v.json 2>&1
done
KVT_LIB=libkvt_mb6.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "append" > gpurun_out/mb6_pytest.log 2>&1; echo "exit $?" >> gpurun_out/mb6_pytest.log
bash tools/gpu_bench_ab.sh mbb llama-3.25 "KVT_LIB=libkvt.so;KVT_LIB=libkvt_mb6.so;KVT_LIB=libkvt_mb8.so"

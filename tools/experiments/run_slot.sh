mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_slot.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_slot.log
: > gpurun_out/slot.log
for cfg in "--kb 4 --vb 2" "--kb 2 --vb 2" "--kb 8 --vb 4" "--kb 4 --vb 4" "--kb 4 --vb 4 --g 7 --H 4"; do
  timeout 300 python tools/kbench.py $cfg --reps 50 >> gpurun_out/slot.log 2>&1
done
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_slot.json 2>&1

#!/bin/bash
# Round-2 final record (run via gpurun): full -m gpu suite, smoke, bench lines of every workload, launch list,
# ncu --set full of the dominant kernel (K4V2, Llama shape) and of the Qwen KV4 (g = 7) kernel.
mkdir -p gpurun_out /tmp/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/fin_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/fin_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/fin_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/fin_smoke.log
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/fin_bench_llama-3.25.log 2>&1; echo "exit $?" >> gpurun_out/fin_bench_llama-3.25.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --paged > gpurun_out/fin_bench_llama-3.25-paged.log 2>&1
for w in llama-kv8 qwen-4.00 qwen-4.00-pertoken qwen-3.92 llama-128k-seqshard; do
  timeout 900 python bench.py --steps 30 --warmup 5 --workload $w --no-cpu-baseline > gpurun_out/fin_bench_$w.log 2>&1; echo "exit $?" >> gpurun_out/fin_bench_$w.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|combine|append" -s 100 -c 200 --csv --log-file gpurun_out/fin_launches.csv python bench.py --profile --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/fin_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mma -s 3 -c 1 -o /tmp/prof/fin_K4V2 -f python tools/kbench.py --kb 4 --vb 2 --reps 1 > gpurun_out/fin_ncu_K4V2.log 2>&1
ncu -i /tmp/prof/fin_K4V2.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/fin_K4V2.source.csv.gz
python tools/ncu_summary.py /tmp/prof/fin_K4V2.ncu-rep > gpurun_out/fin_K4V2.summary.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:decode_mma -s 3 -c 1 -o /tmp/prof/fin_qwen -f python tools/kbench.py --kb 4 --vb 4 --g 7 --H 4 --reps 1 > gpurun_out/fin_ncu_qwen.log 2>&1
python tools/ncu_summary.py /tmp/prof/fin_qwen.ncu-rep > gpurun_out/fin_qwen.summary.txt 2>&1

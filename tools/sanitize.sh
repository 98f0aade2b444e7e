#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py (logs -> gpurun_out/sanitize_*.log)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.log
done
# the per-SM plan's unclaimed-item path (every 3rd CTA gives up its item; the last CTA runs them)
for tool in memcheck racecheck synccheck; do
  KVT_SMPLAN_DROP=3 KVT_SAN_ONLY=smplan timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_smplan_drop.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}_smplan_drop.log
done

#!/bin/bash
# bench A/B over environment switches:  bash tools/gpu_bench_ab.sh TAG WORKLOAD "ENV1=.. ENV2=..;ENV1=..;..."
mkdir -p gpurun_out
tag=$1; wl=$2; IFS=';' read -ra VS <<< "$3"
: > gpurun_out/${tag}_benchab.log
for v in "${VS[@]}"; do
  env $v timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_tmp.log 2>&1
  echo "== $v" >> gpurun_out/${tag}_benchab.log
  python - gpurun_out/${tag}_tmp.log >> gpurun_out/${tag}_benchab.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        print(f"value {d['value']:.0f} ms/step {d['ms_per_step']:.4f} frac {r['frac']:.4f} clocks {d.get('clocks', {}).get('sm_mhz')}")
        for k, v in sorted(r.get("by_pair", {}).items()):
            print(f"   {k:8s} x{v['layers']:2d} {v['us_per_launch']:7.1f} us  frac {v['frac']:.3f}")
PY
  tail -2 gpurun_out/${tag}_tmp.log | grep -i error >> gpurun_out/${tag}_benchab.log
done

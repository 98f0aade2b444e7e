mkdir -p gpurun_out
: > gpurun_out/fill.log
for B in 55 64 74; do timeout 300 python tools/kbench.py --kb 4 --vb 2 --B $B >> gpurun_out/fill.log 2>&1; done
for B in 64 74; do KVT_NCTA=592 timeout 300 python tools/kbench.py --kb 4 --vb 2 --B $B >> gpurun_out/fill.log 2>&1; done

mkdir -p gpurun_out
: > gpurun_out/ncta2.log
run() { echo "NCTA=$1 $2" >> gpurun_out/ncta2.log; if [ $1 == 0 ]; then timeout 300 python tools/kbench.py $2 >> gpurun_out/ncta2.log 2>&1; else KVT_NCTA=$1 timeout 300 python tools/kbench.py $2 >> gpurun_out/ncta2.log 2>&1; fi; }
run 0 "--kb 4 --vb 2 --B 32"; run 256 "--kb 4 --vb 2 --B 32"
run 0 "--kb 4 --vb 2 --B 16"; run 128 "--kb 4 --vb 2 --B 16"
run 0 "--kb 4 --vb 2 --B 20"; run 160 "--kb 4 --vb 2 --B 20"
run 0 "--kb 4 --vb 4 --g 7 --H 4 --B 32"; run 128 "--kb 4 --vb 4 --g 7 --H 4 --B 32"
run 0 "--kb 4 --vb 4 --g 7 --H 4 --B 40"; run 160 "--kb 4 --vb 4 --g 7 --H 4 --B 40"
run 0 "--kb 4 --vb 4 --g 7 --H 4 --B 100"; run 400 "--kb 4 --vb 4 --g 7 --H 4 --B 100"
run 0 "--kb 8 --vb 4 --B 64"; run 512 "--kb 8 --vb 4 --B 64"

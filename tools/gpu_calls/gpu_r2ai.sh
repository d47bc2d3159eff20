cd tools/micro
timeout 120 ./tdisp_bench 0.05 > ../../gpurun_out/tdisp_005.txt 2>&1; echo t=$?
timeout 120 ./tdisp_bench 0.01 > ../../gpurun_out/tdisp_001.txt 2>&1
timeout 120 ./tdisp_bench 0.1 > ../../gpurun_out/tdisp_010.txt 2>&1

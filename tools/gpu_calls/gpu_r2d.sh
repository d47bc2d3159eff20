timeout 120 tools/micro/tmem_bench > gpurun_out/tmem_bench.txt 2>&1; echo tmem=$?

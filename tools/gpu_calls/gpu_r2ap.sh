timeout 120 tools/micro/bulk_bench > gpurun_out/bulk_bench.txt 2>&1; echo b=$?

cd tools/micro
timeout 120 ./pm_bench 0.05 > ../../gpurun_out/pm_005.txt 2>&1; echo pm=$?
timeout 120 ./pm_bench 0.01 > ../../gpurun_out/pm_001.txt 2>&1
timeout 120 ./scan_bench 0.05 > ../../gpurun_out/scan_005.txt 2>&1; echo scan=$?

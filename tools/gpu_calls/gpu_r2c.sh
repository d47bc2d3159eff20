cd tools/micro
for r in 0.05 0.01 0.1; do ./scan_bench3 $r; done > ../../gpurun_out/scan_bench3.txt 2>&1; echo scan=$?

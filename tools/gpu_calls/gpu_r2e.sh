cd tools/micro
for r in 0.05 0.01; do timeout 120 ./scan_bench4 $r; done > ../../gpurun_out/scan_bench4.txt 2>&1; echo scan=$?

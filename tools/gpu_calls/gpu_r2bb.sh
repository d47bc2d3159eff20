cd tools/micro
for r in 0.05 0.01 0.1; do timeout 120 ./sd_bench $r > ../../gpurun_out/sd_$r.txt 2>&1; done; echo ok

cd tools/micro
for r in 0.05 0.01 0.1 0.02; do timeout 120 ./solo_bench $r > ../../gpurun_out/solo_$r.txt 2>&1; done; echo ok

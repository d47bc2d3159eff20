cd tools/micro
for r in 0.05 0.01; do timeout 120 ./pair_bench $r > ../../gpurun_out/pair_$r.txt 2>&1; done; echo ok

nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd tools/micro
for r in 0.05 0.01 0.1; do ./scan_bench $r; done > ../../gpurun_out/scan_bench.txt 2>&1; echo scan=$?
cd ../..
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep > gpurun_out/bench0.log 2>&1; echo bench=$?

timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo bench_c5=$?

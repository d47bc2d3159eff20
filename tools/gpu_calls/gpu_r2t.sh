timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cudnn.log 2>&1; echo bench=$?
timeout 900 python bench.py --config C4a --steps 20 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/bench_cudnn_c4a.log 2>&1; echo bench=$?

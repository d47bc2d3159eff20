timeout 600 python -m pytest tests/test_gpu_auto.py -q -x > gpurun_out/pytest_auto_shfl.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_shfl.log 2>&1; echo bench=$?

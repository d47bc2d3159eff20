timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo bench_c5=$?

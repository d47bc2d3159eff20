timeout 1500 python -m pytest tests/test_gpu_bench.py -q -x > gpurun_out/pytest_bench.log 2>&1; echo pytest=$?
SC_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_2rank_shared.log 2>&1; echo b2=$?

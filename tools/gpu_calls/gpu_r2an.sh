timeout 900 python -m pytest tests/test_gpu_backward.py -q -x > gpurun_out/pytest_bwd.log 2>&1; echo pytest=$?
timeout 600 python bench.py --backward --steps 20 --warmup 3 > gpurun_out/bench_bwd_new.log 2>&1; echo bwd=$?

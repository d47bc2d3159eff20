timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest=$?
timeout 600 python bench.py --backward --steps 20 --warmup 3 > gpurun_out/bench_bwd_final.log 2>&1; echo bwd=$?

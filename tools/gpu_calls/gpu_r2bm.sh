timeout 1800 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_fuzz.py -q -x -k "table2 or fuzz or jit or forced or integer" > gpurun_out/pytest_1x1.log 2>&1; echo pytest=$?
timeout 900 python bench.py --table2 > gpurun_out/table2_1x1.log 2>&1; echo t2=$?

timeout 1800 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_fuzz.py tests/test_gpu_nonfinite.py tests/test_gpu_auto.py tests/test_gpu_chain.py -q -x > gpurun_out/pytest_1x1.log 2>&1; echo pytest=$?
timeout 900 python bench.py --table2 > gpurun_out/table2_1x1.log 2>&1; echo t2=$?

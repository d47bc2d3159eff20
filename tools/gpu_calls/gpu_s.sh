timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --table2 > gpurun_out/table2.log 2>&1; echo table2=$?

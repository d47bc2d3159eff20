timeout 600 python -m pytest tests/test_gpu_auto.py -q -x > gpurun_out/pytest_auto_head.log 2>&1; echo pytest=$?

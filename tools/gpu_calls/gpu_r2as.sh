timeout 900 python -m pytest tests/test_gpu_backward.py -q -x > gpurun_out/pytest_bwd.log 2>&1; echo pytest=$?
bash tools/gpu_calls/gpu_r2ar.sh new2

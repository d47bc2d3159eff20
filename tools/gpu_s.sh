timeout 900 python -m pytest tests/test_gpu_dense.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/probe_run.py C2 C4a C3 C1 C4b > gpurun_out/probe.log 2>&1; echo probe=$?

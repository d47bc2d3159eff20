timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest=$?
bash tools/gpu_r2_measure.sh > gpurun_out/measure.log 2>&1

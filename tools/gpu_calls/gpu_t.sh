set -x
for v in "C4b 0.5 3 8" "C4b 0.5 3 3" "C4a 0.5 3 8" "C2 0.95 3 8"; do timeout 120 python tools/isolate.py $v; echo "rc=$?"; done > gpurun_out/isolate.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python tools/probe_run.py C2 C4a C3 C1 C4b > gpurun_out/probe.log 2>&1; echo probe=$?

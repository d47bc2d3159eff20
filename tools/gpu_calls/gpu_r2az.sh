timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?

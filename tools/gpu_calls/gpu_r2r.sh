timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_default.log 2>&1; echo ref=$?

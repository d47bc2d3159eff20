timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_batches.py tests/test_gpu_fuzz.py -q -x > gpurun_out/t_c1.log 2>&1; echo "pytest=$?"
timeout 900 python bench.py --config C1 > gpurun_out/bench_C1.jsonl 2> gpurun_out/bench_C1.err; echo "bench=$?"

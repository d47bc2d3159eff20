timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_fuzz.py -q -x > gpurun_out/t_sparse.log 2>&1; echo "pytest=$?"
timeout 600 python bench.py --table2 > gpurun_out/t2.jsonl 2> gpurun_out/t2.err; echo "t2=$?"

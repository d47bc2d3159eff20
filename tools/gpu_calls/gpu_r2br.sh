timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_fuzz.py tests/test_gpu_backward.py -q -x > gpurun_out/t_sparse.log 2>&1; echo "pytest=$?"
timeout 900 python tools/jit_1x1_probe.py 0.9 > gpurun_out/j1x1_all.txt 2>&1; echo "probe=$?"
timeout 600 python bench.py --table2 > gpurun_out/t2.jsonl 2> gpurun_out/t2.err; echo "t2=$?"

timeout 900 python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err; echo "bench=$?"
timeout 1200 python -m pytest tests/test_gpu_bench.py -q -x > gpurun_out/t_bench.log 2>&1; echo "pytest=$?"

timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_auto.py -q -x > gpurun_out/t_dense.log 2>&1; echo "pytest=$?"
timeout 900 python bench.py --no-sweep --no-cpu-baseline > gpurun_out/bench_dsplit.jsonl 2> gpurun_out/bench_dsplit.err; echo "bench=$?"
SC_DENSE_SPLIT=0 timeout 900 python bench.py --no-sweep --no-cpu-baseline > gpurun_out/bench_dnosplit.jsonl 2> gpurun_out/bench_dnosplit.err; echo "bench0=$?"
timeout 900 python bench.py --config C4a --no-sweep --no-cpu-baseline > gpurun_out/bench_dsplit4a.jsonl 2> gpurun_out/bench_dsplit4a.err; echo "bench4a=$?"

timeout 900 python -m pytest tests/test_gpu_batches.py -q -x > gpurun_out/t_hb.log 2>&1; echo "pytest=$?"
timeout 900 python bench.py --no-sweep --no-cpu-baseline > gpurun_out/bench_hb.jsonl 2> gpurun_out/bench_hb.err; echo "bench=$?"

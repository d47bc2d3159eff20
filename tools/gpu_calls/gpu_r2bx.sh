timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_fuzz.py tests/test_gpu_chain.py tests/test_gpu_batches.py -q -x > gpurun_out/t_emit.log 2>&1; echo "pytest=$?"
for c in C2 C4a; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_e_$c.jsonl 2> gpurun_out/bench_e_$c.err; echo "bench $c=$?"; done

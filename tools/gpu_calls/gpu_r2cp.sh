timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_batches.py -q -x > gpurun_out/t_sort2.log 2>&1; echo "pytest=$?"
for c in C2 C4a C4b C3 C1; do SC_SORT_STREAMS=1 timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_sortb_$c.jsonl 2> gpurun_out/bench_sortb_$c.err; echo "bench $c $?"; done

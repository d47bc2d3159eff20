timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_backward.py -q -x > gpurun_out/t_cnt.log 2>&1; echo "pytest=$?"
for c in C4a C3 C2 C4b; do timeout 900 python bench.py --config $c --no-sweep --no-cpu-baseline > gpurun_out/bench_cnt_$c.jsonl 2> gpurun_out/bench_cnt_$c.err; echo "bench $c=$?"; done

timeout 1500 python -m pytest tests/test_gpu_sparse.py -q -x -k "full_config or small_batch" > gpurun_out/t_em6.log 2>&1; echo "pytest=$?"
for c in C2 C4a; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_em6_$c.jsonl 2> gpurun_out/bench_em6_$c.err; echo "bench $c=$?"; done

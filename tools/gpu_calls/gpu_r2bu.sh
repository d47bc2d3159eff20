timeout 900 python -m pytest tests/test_gpu_chain.py -q -x > gpurun_out/t_chain.log 2>&1; echo "pytest=$?"
for k in 1 2 4 8; do SC_CHAIN_CHUNKS=$k timeout 900 python bench.py --config C5 --no-cpu-baseline > gpurun_out/bench_C5_k$k.jsonl 2> gpurun_out/bench_C5_k$k.err; echo "c5 k=$k $?"; done

timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_gpu_all.log 2>&1; echo "pytest=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err; echo "bench=$?"
for c in C1 C3 C4a C4b C4 C5; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.jsonl 2> gpurun_out/bench_$c.err; echo "bench $c=$?"; done
timeout 900 python bench.py --table2 > gpurun_out/t2.jsonl 2> gpurun_out/t2.err; echo "t2=$?"

timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_ord.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ord2_c2.log 2>&1; echo bench=$?
for c in C3 C4a C4b; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/bench_ord2_$c.log 2>&1; echo bench_$c=$?; done
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ord2_C5.log 2>&1; echo c5=$?

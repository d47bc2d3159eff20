timeout 900 python -m pytest tests -m gpu -q -x -k "sparse or chain or auto or nonfinite" > gpurun_out/pytest_pdl.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pdl.log 2>&1; echo bench=$?
for c in C3 C4a C4b; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/bench_pdl_$c.log 2>&1; echo bench_$c=$?; done

timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_newvar.log 2>&1; echo pytest=$?
for c in C1 C4a C4b C4; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_newvar_$c.log 2>&1; echo bench_$c=$?; done

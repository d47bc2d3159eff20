timeout 900 python -m pytest tests -m gpu -q -x -k "chain or fuzz or sparse or nonfinite" > gpurun_out/pytest_sh.log 2>&1; echo pytest=$?
for c in C2 C4a C4b; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/bench_sh_$c.log 2>&1; echo bench_$c=$?; done

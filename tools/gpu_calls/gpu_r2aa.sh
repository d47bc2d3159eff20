timeout 900 python -m pytest tests -m gpu -q -x -k "sparse or chain or fuzz or nonfinite" > gpurun_out/pytest_ch8.log 2>&1; echo pytest=$?
for c in C4b C1 C4; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/bench_ch8_$c.log 2>&1; echo bench_$c=$?; done

timeout 900 python -m pytest tests -m gpu -q -x -k "sparse or chain or fuzz or auto or nonfinite" > gpurun_out/pytest_gpu_s1.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_s1.log 2>&1; echo bench=$?
for c in C4a C4b C3 C1; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/bench_${c}_s1.log 2>&1; echo bench_$c=$?; done

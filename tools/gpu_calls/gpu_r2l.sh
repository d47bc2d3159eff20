timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_split_c2.log 2>&1; echo bench=$?
for c in C4a; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/bench_split_$c.log 2>&1; echo bench_$c=$?; done

timeout 900 python -m pytest tests -m gpu -q -x -k "sparse or chain or fuzz or auto or nonfinite or backward" > gpurun_out/pytest_seg.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_seg_c2.log 2>&1; echo bench=$?
for c in C3 C4a C4b C1; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/bench_seg_$c.log 2>&1; echo bench_$c=$?; done
for c in C2 C4a; do
python tools/prof_run.py $c 0.95 2 > gpurun_out/plain_$c.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:compact --csv --log-file gpurun_out/compact_launches4_$c.csv python tools/prof_run.py $c 0.95 2 > gpurun_out/ncu_$c.log 2>&1; echo ncu_$c=$?
done

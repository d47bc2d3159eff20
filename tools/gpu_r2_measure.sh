# Round-2 measurement pass (one B200): bench lines for every config, the reference arm,
# FFMA/FFMA2 census, launch list, ncu captures of the gather and the dense kernel.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out/m
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/m/bench_C2.log 2>&1; echo bench_C2=$?
for c in C1 C3 C4a C4b C4; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/m/bench_$c.log 2>&1; echo bench_$c=$?
done
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/m/bench_C5.log 2>&1; echo bench_C5=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/m/bench_ref.log 2>&1; echo ref=$?
python tools/fma_census.py gpurun_out/m/fma_counts_plain.jsonl > gpurun_out/m/fma_plain.log 2>&1 && \
ncu --metrics smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,gpu__time_duration.sum \
    --clock-control none -k regex:gather_fast --csv --log-file gpurun_out/m/fma_census.csv \
    python tools/fma_census.py gpurun_out/m/fma_counts.jsonl > gpurun_out/m/fma_ncu.log 2>&1; echo fma=$?
python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/m/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/m/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/m/ncu_launch.log 2>&1; echo launches=$?
python tools/prof_run.py C2 0.95 1 > gpurun_out/m/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gather_fast -c 1 -o gpurun_out/m/gather_C2 python tools/prof_run.py C2 0.95 1 > gpurun_out/m/ncu_gather.log 2>&1; echo ncu_gather=$?
python tools/dense_probe.py > gpurun_out/m/plain_dense.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dense_tc -c 1 -o gpurun_out/m/dense_C2 python tools/dense_probe.py > gpurun_out/m/ncu_dense.log 2>&1; echo ncu_dense=$?
timeout 900 python bench.py --table2 > gpurun_out/m/table2.log 2>&1; echo table2=$?
timeout 600 python bench.py --backward --steps 20 --warmup 3 > gpurun_out/m/bench_bwd.log 2>&1; echo bwd=$?
timeout 300 python tools/crossover_curve.py C2 C4a C4b > gpurun_out/m/crossover.txt 2>&1; echo crossover=$?
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/m/smoke.log 2>&1; echo smoke=$?

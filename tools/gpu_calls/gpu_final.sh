set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo bench_c5=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
python tools/prof_run.py C2 0.95 1 > gpurun_out/plain_prof.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gather_fast -c 1 -o gpurun_out/gather_full python tools/prof_run.py C2 0.95 1 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
python tools/prof_run.py C2 0.95 1 > gpurun_out/plain_prof2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:compact -c 2 -o gpurun_out/compact_full python tools/prof_run.py C2 0.95 1 > gpurun_out/ncu_compact.log 2>&1; echo ncucompact=$?
python tools/dense_probe.py > gpurun_out/plain_dense.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:dense_tc -c 1 -o gpurun_out/dense_full python tools/dense_probe.py > gpurun_out/ncu_dense.log 2>&1; echo ncudense=$?
timeout 300 python tools/crossover_curve.py C2 C4a C4b > gpurun_out/crossover.txt 2>&1; echo crossover=$?
timeout 300 python tools/auto_overhead.py > gpurun_out/auto_overhead.txt 2>&1; echo auto=$?
timeout 300 python bench.py --backward --steps 20 --warmup 3 > gpurun_out/bench_bwd.log 2>&1; echo bwd=$?

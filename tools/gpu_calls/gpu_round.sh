set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
timeout 600 python tools/prof_run.py C2 0.95 2 dense > gpurun_out/prof.log 2>&1; echo prof=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_fast -c 1 -o gpurun_out/gather_full python tools/prof_run.py C2 0.95 1 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense -c 1 -o gpurun_out/dense_full python tools/prof_run.py C2 0.95 1 dense > gpurun_out/ncu_dense.log 2>&1; echo ncudense=$?

timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu-baseline > gpurun_out/b_short.log 2>&1; echo "short=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu=$?"

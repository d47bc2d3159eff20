timeout 900 python -m pytest tests -m gpu -q -x -k "chain or fuzz or sparse" > gpurun_out/pytest_rows.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rows_C5.log 2>&1; echo c5=$?
python tools/chain_run.py 1024 > gpurun_out/plain_chain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/chain_launches2.csv python tools/chain_run.py 1024 > gpurun_out/ncu_chain.log 2>&1; echo ncu=$?

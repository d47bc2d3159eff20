timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_solo.log 2>&1; echo pytest=$?
for c in C2 C1 C3 C4a C4b; do
timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/solo_$c.log 2>&1; echo $c=$?
done

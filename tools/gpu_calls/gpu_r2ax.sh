timeout 900 python -m pytest tests/test_gpu_sparse.py -q -x > gpurun_out/pytest_fused_sparse.log 2>&1; echo sparse=$?
for c in C2 C1; do
timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/fb_$c.log 2>&1; echo $c=$?
SC_NO_FUSED=1 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/fb0_$c.log 2>&1; echo ${c}0=$?
done

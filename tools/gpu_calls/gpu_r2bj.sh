timeout 2400 python tools/fuzz_sweep.py 6 30 10 > gpurun_out/fuzz_sweep2.txt 2>&1; echo fuzz=$?

timeout 2400 python tools/fuzz_sweep.py 4 30 > gpurun_out/fuzz_sweep.log 2>&1; echo sweep=$?

timeout 2400 python tools/bwd_fuzz.py 80 1 > gpurun_out/bwd_fuzz.txt 2>&1; echo fuzz=$?

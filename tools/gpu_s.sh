timeout 600 python tools/variant_sweep.py C2 0.95,0.99 "21 34 35" > gpurun_out/sweep.log 2>&1; echo sweep=$?

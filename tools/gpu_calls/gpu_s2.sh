timeout 600 python tools/variant_sweep.py C2 0.95,0.99 "12 90 91" > gpurun_out/sweep.log 2>&1; echo sweep=$?

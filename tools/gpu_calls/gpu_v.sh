timeout 600 python tools/variant_sweep.py "$@" > gpurun_out/sweep.log 2>&1; echo sweep=$?

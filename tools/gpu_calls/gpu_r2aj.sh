timeout 300 python tools/tm_probe.py 60 C2 0.9 0.95 0.99 > gpurun_out/tm_probe.txt 2>&1; echo probe=$?

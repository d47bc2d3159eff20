timeout 300 python tools/tm_probe.py 63 C2 0.95 0.99 > gpurun_out/tm_probe_63_nocp.txt 2>&1; echo probe=$?

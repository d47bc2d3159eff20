python tools/bwd_probe.py 0.95 > gpurun_out/bwdp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bwd_kernel -c 2 -o gpurun_out/bwd_C2 python tools/bwd_probe.py 0.95 > gpurun_out/ncu_bwd.log 2>&1; echo ncu=$?

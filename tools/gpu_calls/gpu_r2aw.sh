python tools/prof_run.py C2 0.95 1 > gpurun_out/pf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gather_fused -c 1 -o gpurun_out/fused_C2 python tools/prof_run.py C2 0.95 1 > gpurun_out/ncu_fused.log 2>&1; echo ncu=$?

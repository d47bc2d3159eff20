export SC_FORCE_VARIANT=12
python tools/prof_run.py C2 0.95 1 > gpurun_out/plain_c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:compact_plane -c 2 -o gpurun_out/cplane python tools/prof_run.py C2 0.95 1 > gpurun_out/ncu_cplane.log 2>&1; echo ncu=$?

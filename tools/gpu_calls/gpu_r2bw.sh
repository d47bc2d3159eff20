python tools/stage1_probe.py C2 0.95 2 > gpurun_out/s1.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:compact_plane -c 2 -o gpurun_out/s1_C2 python tools/stage1_probe.py C2 0.95 2 > gpurun_out/s1_ncu.log 2>&1; echo "ncu=$?"
ncu --set full --clock-control none --import-source on -k regex:compact_plane -c 2 -o gpurun_out/s1_C4a python tools/stage1_probe.py C4a 0.95 2 > gpurun_out/s1_ncu4.log 2>&1; echo "ncu4=$?"

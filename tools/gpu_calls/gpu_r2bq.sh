timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -x -k "jit" > gpurun_out/t_jit.log 2>&1; echo "pytest=$?"
timeout 900 python tools/jit_1x1_probe.py 0.9 "512,14,256;528,14,256;480,14,208;512,14,224" "1,8,11,1,32,2,2,254;1,8,11,1,32,3,3,254;1,8,11,1,32,2,3,254" > gpurun_out/j1x1_w14.txt 2>&1; echo "w14=$?"
timeout 900 python tools/jit_1x1_probe.py 0.9 "832,7,384;1024,7,512;832,7,320" "1,6,11,1,32,3,2,510;1,6,11,1,32,2,2,254;1,8,11,1,32,3,3,254" > gpurun_out/j1x1_w7.txt 2>&1; echo "w7=$?"

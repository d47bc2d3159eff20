for v in 1,2,7,2,16,2,2,126 1,2,7,2,16,2,3,126 1,2,7,2,8,3,2,126 2,1,7,2,16,2,2,126 3,1,7,2,16,2,2,126 1,2,5,2,16,2,2,126 2,1,5,2,16,2,2,126; do
timeout 300 python tools/tm_probe.py jit:$v C4a 0.95 > "gpurun_out/minb_C4a_$v.txt" 2>&1; echo C4a$v=$?
done
for v in 2,2,7,2,16,2,2,126 3,2,7,2,16,2,2,126 1,4,7,2,16,2,2,126 1,4,7,2,8,3,2,126 2,2,5,2,16,2,2,126 4,1,7,2,16,2,2,126; do
timeout 300 python tools/tm_probe.py jit:$v C2 0.95 > "gpurun_out/minb_C2_$v.txt" 2>&1; echo C2$v=$?
done

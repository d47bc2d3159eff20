for v in jit:2,4,11,1,16,2,3,254 jit:2,4,11,1,8,4,3,254 jit:2,4,11,1,12,3,3,254 jit:2,4,11,1,8,3,3,254 jit:2,4,11,1,4,8,3,254; do
timeout 300 python tools/tm_probe.py $v C2 0.95 0.99 > "gpurun_out/ring_$v.txt" 2>&1; echo $v=$?
done

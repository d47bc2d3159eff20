for v in jit:1,4,15,1,16,2,2,254 jit:1,4,14,1,16,2,2,254 jit:1,4,15,1,12,2,3,254 jit:1,4,13,1,16,2,3,254 jit:1,4,11,1,16,2,3,254; do
timeout 300 python tools/tm_probe.py $v C2 0.95 0.99 > "gpurun_out/ty1_C2_$v.txt" 2>&1; echo $v=$?
done

for v in 62 63 64 jit:2,4,11,1,16,2,8,62; do
timeout 300 python tools/tm_probe.py $v C2 0.9 0.95 0.99 > gpurun_out/tm_probe_$v.txt 2>&1; echo probe$v=$?
done
timeout 300 python tools/tm_probe.py 62 C2:512 0.95 0.99 > gpurun_out/tm_probe_62_512.txt 2>&1; echo p=$?

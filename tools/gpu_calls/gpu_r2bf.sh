# NW=13 compute warps (14 per CTA, <= 146 registers): fewer rounds for C4a / C3 / C5-like grids
for v in jit:2,2,13,1,32,2,3,254 jit:2,2,13,1,16,2,3,254 jit:2,2,11,1,32,2,3,254 jit:1,4,13,1,16,2,3,254; do
timeout 300 python tools/tm_probe.py $v C4a 0.95 0.99 > "gpurun_out/nw13_C4a_$v.txt" 2>&1; echo C4a$v=$?
done
for v in jit:3,1,13,1,16,2,3,254 jit:3,1,11,1,16,2,3,254; do
timeout 300 python tools/tm_probe.py $v C3 0.95 > "gpurun_out/nw13_C3_$v.txt" 2>&1; echo C3$v=$?
done
for v in jit:2,4,13,1,16,2,3,254 jit:2,4,13,1,8,3,3,254; do
timeout 300 python tools/tm_probe.py $v C2:1024 0.95 > "gpurun_out/nw13_C2_$v.txt" 2>&1; echo C2$v=$?
done

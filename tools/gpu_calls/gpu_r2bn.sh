p() { timeout 300 python tools/tm_probe.py "$1" "$2" "$3" > "gpurun_out/kl8_$2_$1.txt" 2>&1; echo "$2 $1=$?"; }
p jit:1,8,11,1,16,2,3,254 T2.GoogLeNet-Inception4a.1 0.9
p jit:2,8,11,1,16,2,3,254 T2.GoogLeNet-Inception4a.1 0.9
p jit:2,8,11,1,16,2,3,254 T2.GoogLeNet-Inception5a.1 0.95
p jit:1,8,11,1,32,2,3,254 T2.GoogLeNet-Inception5a.1 0.95
p jit:2,8,11,1,16,2,3,254 T2.GoogLeNet-Inception5a.2 0.9
p jit:1,8,11,1,16,2,3,254 T2.GoogLeNet-Inception4a.2 0.9
p jit:2,6,11,1,16,2,3,254 T2.GoogLeNet-Inception4a.1 0.9

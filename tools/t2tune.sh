for l in LeNet-Conv2 AlexNetC-Conv3 AlexNetI-Conv4 GoogLeNet-Inception4a.1 GoogLeNet-Inception4a.2 GoogLeNet-Inception4e.3 GoogLeNet-Inception5a.1 GoogLeNet-Inception5a.2 GoogLeNet-Inception5b.3 GoogLeNet-Inception5b.5; do
  s=0.9; case $l in LeNet-Conv2|GoogLeNet-Inception5a.1|GoogLeNet-Inception5b.3|GoogLeNet-Inception5b.5) s=0.95;; esac
  timeout 300 python tools/jit_tune.py T2:$l $s quick > gpurun_out/t2_$l.log 2>&1
  echo "== $l"; head -1 gpurun_out/t2_$l.log; grep -A3 "best" gpurun_out/t2_$l.log | tail -3
done

tag=${1:-new}
for c in C2 C1 C3 C4a C4b; do
timeout 600 python bench.py --backward --config $c --steps 5 --warmup 3 > gpurun_out/bwd_${tag}_$c.log 2>&1; echo $c=$?
done

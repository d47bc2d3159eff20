timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > gpurun_out/t_bwd.log 2>&1; echo "pytest=$?"
timeout 900 python bench.py --backward > gpurun_out/bwd_C2.jsonl 2> gpurun_out/bwd_C2.err; echo "bwd=$?"
for c in C4a C3; do timeout 900 python bench.py --backward --config $c > gpurun_out/bwd_$c.jsonl 2> gpurun_out/bwd_$c.err; echo "bwd $c=$?"; done

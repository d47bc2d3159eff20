for c in C2 C1 C3 C4a C4b; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.jsonl 2> gpurun_out/bench_$c.err; echo "bench $c=$?"; done

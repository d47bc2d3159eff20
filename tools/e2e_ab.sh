for i in 1 2; do
for cfg in "2 8" "1 4"; do set -- $cfg
SC_HOST_STREAMS=$1 SC_HOST_CHUNKS=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-sweep --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('streams=$1 chunks=$2', d['value'], e['ms_per_step'], e['ms_mean'])"
done; done

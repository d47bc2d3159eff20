#!/bin/bash
# time the stage-2 variants that match a config: tools/variant_timing.sh C2 "1 6 0"
cfg=${1:-C2}; vars=${2:-"1 6"}
for v in $vars; do
  SC_FORCE_VARIANT=$v python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('variant', d['config']['variant'], 'gather_us', d['stages_us'], 'ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'sweep', {k:(v['gather_us']) for k,v in d['sweep'].items()})
"
done

#!/bin/bash
# bench one config and print value + per-level GS / restriction ms (A/B helper)
CFG=${1:-4}
python bench.py --config $CFG --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
b=d['breakdown_ms']
print(round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'gs', {l:v['ms'] for l,v in b['gs_sweep'].items()}, 'rr', {l:v['ms'] for l,v in b['residual_restrict'].items()}, 'asm', b.get('assembly',{}).get('0',{}).get('ms'), 'ms/step', round(d['ms_per_step'],3))
"

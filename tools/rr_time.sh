#!/bin/bash
# bench one config; print value, restriction+residual ms per level and assembly ms (A/B helper)
CFG=${1:-4}
python bench.py --config $CFG --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
b=d['breakdown_ms']
print(round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'rr', {l:v['ms'] for l,v in b['residual_restrict'].items()}, 'asm', b['assembly'], 'gal', round(sum(v['ms'] for v in b['galerkin'].values()),3))
"

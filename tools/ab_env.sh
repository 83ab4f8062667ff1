#!/bin/bash
# A/B of environment switches on bench.py: tools/ab_env.sh "<bench args>" "ENV=..." "ENV=..." ...
args="$1"; shift
for e in "$@"; do
  env $e timeout 600 python bench.py --no-cpu-baseline $args > gpurun_out/abenv.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/abenv.json'));kb=d['kernel_breakdown']
print('$e', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None, 'fwd', round(kb['blend_forward']['ms_per_step']*1000,1), 'bwd', round(kb['blend_backward']['ms_per_step']*1000,1))"
done

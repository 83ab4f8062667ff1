#!/bin/bash
# A/B per-kernel timing of library variants: tools/ab_kernels.sh <regex> <variant> ... ("base" = product lib)
re="$1"; shift
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="SPLAT_B200_LIB=paper_2411_12788_b200/lib_$v/libsplat_b200.so"; fi
  env $lib timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 200 --warmup 20 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json,re;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['value'],1), {k:round(x['ms_per_step']*1000,1) for k,x in d['kernel_breakdown'].items() if re.search('$re',k)})"
done

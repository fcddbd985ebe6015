#!/bin/bash
# Round-trip tuning variants (DCTADJ_RT_VARIANT, tuning-build library) on the given configs:
#   LIB=tools/bin/libdctadj_tune.so VARIANTS="0 1 2 3 4" tools/rt_variants.sh c3_pre c3_post c2
for c in "$@"; do
  for v in ${VARIANTS:-0 1 2 3 4}; do
    DCTADJ_RT_VARIANT=$v DCTADJ_LIB=$PWD/$LIB python bench.py --config $c --no-per-config --no-cpu --steps 20 --warmup 5 2>/dev/null |
      python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$c variant $v', round(d['value']/1e9,1), 'G coef/s frac', round(r['frac'],3), {k:round(x,4) for k,x in r['per_launch_ms'].items()}, 'gate', d['config'].get('gate_max_rel_err_all_ranks'))
"
  done
done

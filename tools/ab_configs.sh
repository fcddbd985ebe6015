#!/bin/bash
# A/B of several libraries on the same box, interleaved:
#   LIBS="tools/bin/a.so tools/bin/b.so" REPS=2 tools/ab_configs.sh <configs...>
# prints value / roofline fraction / per-launch ms per config and library
LIBS=${LIBS:-paper_2505_23618_b200/libdctadj.so}
for rep in $(seq ${REPS:-2}); do
  for c in "$@"; do
    for lib in $LIBS; do
      DCTADJ_LIB=$PWD/$lib python bench.py --config $c --no-per-config --no-cpu --steps 20 --warmup 5 2>/dev/null |
        python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$c', '$lib'.split('/')[-1], round(d['value']/1e9,1), 'G coef/s frac', round(r['frac'],3), {k:round(v,4) for k,v in r['per_launch_ms'].items()}, 'gate', d['config'].get('gate_max_rel_err_all_ranks'))
"
    done
  done
done

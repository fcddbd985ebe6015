#!/bin/bash
# config-4 band-pre timing per tuning variant (DCTADJ_VARIANT; 0 = default, 1-6 = tools/gen_instances.py EXPERIMENT)
for c in c4_dst7_pre c4_dct8_pre; do
  for v in "$@"; do
    DCTADJ_VARIANT=$v timeout 200 python bench.py --config $c --no-cpu --steps 20 --warmup 3 > gpurun_out/v.log 2>&1
    tail -1 gpurun_out/v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', $v, round(d['value']/1e9,1), round(d['roofline']['frac'],3), d['config']['oracle_gate_rel_err'], d['roofline']['per_launch_ms'])" 2>/dev/null || (echo "$c $v FAILED"; tail -3 gpurun_out/v.log)
  done
done

#!/bin/bash
# A/B of the ring-kernel stage hand-off (profiles/r02_tuning.md): tools/ring_stress.py per
# ring tuning variant with two ring-only DCTADJ_TUNING libraries at tools/bin/libdctadj_ring_{fix,old}.so
out=gpurun_out/ring.log; : > $out
for lib in fix old; do
  for v in 0 7 8 9; do
    for op in sub8 band6; do
      echo -n "lib=$lib v=$v " >> $out
      DCTADJ_LIB=tools/bin/libdctadj_ring_$lib.so DCTADJ_VARIANT=$v timeout 120 python tools/ring_stress.py $op 8 >> $out 2>&1 || echo "rc=$? (timeout/hang or error) op=$op" >> $out
    done
  done
done

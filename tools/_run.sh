for v in 0 9 10 11 0; do echo "v$v"; DCTADJ_RT_VARIANT=$v timeout 300 python tools/prof_rt.py 100; done > gpurun_out/prof_rt_hints.log 2>&1

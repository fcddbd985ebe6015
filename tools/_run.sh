for v in 0 1 2 3 4 5 6; do DCTADJ_RT_VARIANT=$v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_rt$v.log 2>&1; done
for v in 0 1 2; do echo "variant $v"; DCTADJ_RT_VARIANT=$v timeout 300 python tools/prof_rt.py 50; done > gpurun_out/prof_rt.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:roundtrip_kernel -s 2 -c 1 -o gpurun_out/rt_full python tools/prof_rt.py 2 > gpurun_out/rt_ncu.log 2>&1

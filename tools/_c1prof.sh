for v in 0 5 8 11; do echo "variant $v"; DCTADJ_VARIANT=$v timeout 120 python tools/prof_c1.py 400; done > gpurun_out/c1_variants3.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_c1.log 2>&1

timeout 600 python bench.py --config c5 --steps 100 --warmup 5 --no-cpu > gpurun_out/cfg_c5.log 2>&1

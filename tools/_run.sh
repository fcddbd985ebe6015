timeout 600 python -m pytest tests -m gpu -x -q -k "host or c2" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench.log 2>&1

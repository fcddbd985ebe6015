timeout 600 python -m pytest tests/test_designer.py tests/test_gpu_parity.py -q -k "designer or descent or optimize or mixed" > gpurun_out/pytest_des.log 2>&1; echo pytest=$? >> gpurun_out/pytest_des.log
timeout 900 python tools/design_gpu.py > gpurun_out/design_gpu.log 2>&1
for c in c3_pre; do timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']/1e9,1), round(d['roofline']['frac'],3), d['roofline']['per_launch_ms'])"; done >> gpurun_out/design_gpu.log 2>&1

timeout 600 python -m pytest tests/test_designer.py -q > gpurun_out/pytest_des.log 2>&1; echo pytest=$? >> gpurun_out/pytest_des.log
timeout 900 python tools/design_gpu.py > gpurun_out/design_gpu.log 2>&1

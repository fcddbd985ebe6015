python tools/diag/copy12.py > gpurun_out/copy12.log 2>&1

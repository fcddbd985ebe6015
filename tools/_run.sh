for r in 1 0; do for c in 8 16 32; do echo "ramp $r"; DCTADJ_HOST_RAMP=$r DCTADJ_HOST_CHUNK_MB=$c timeout 120 python tools/e2e_chunks.py; done; done > gpurun_out/e2e_ramp.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "host" >> gpurun_out/e2e_ramp.log 2>&1

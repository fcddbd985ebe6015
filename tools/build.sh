#!/bin/bash
# Regenerate instantiations and build libdctadj.so; non-zero exit on any failure.
set -e
cd "$(dirname "$0")/.."
python tools/gen_twiddles.py
python tools/gen_instances.py
if ! make -s -j"$(nproc)" -C paper_2505_23618_b200/csrc > /tmp/dctadj_make.log 2>&1; then
  grep -E "error" /tmp/dctadj_make.log | head -20
  echo "BUILD FAILED" >&2
  exit 1
fi
python -c "import ctypes, os; ctypes.CDLL('paper_2505_23618_b200/libdctadj.so', mode=os.RTLD_NOW)"
echo "build ok"

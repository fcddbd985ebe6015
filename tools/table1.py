"""Run the GPU port of the reference's Table-1 benchmark and write the tables.
    python tools/table1.py [out.md]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_23618_b200 import benchmark  # noqa: E402

reps = benchmark.run_benchmark()
out = ["# Table 1 on B200 -- throughput ratio vs the full-matrix transform", "",
       "GPU port of the reference harness (paper_2505_23618_b200/benchmark.py; reference",
       "benchmark.py:130-260): fp32, random-angle adjustments (speed does not depend on",
       "the designed values), oracle-checked, median of 31 CUDA-event samples per cell.",
       "1-D: 4,194,304 vectors per launch (the reference's layout); 2-D: 65,536 32x32 /",
       "16,384 64x64 blocks per launch, one fused kernel per transform.",
       "`dense` is the full-matrix FMA product on the CUDA cores (the paper's baseline, ratio",
       "1.00); `dense_tc` is the same fp32 product on the tensor cores (3xTF32 tcgen05,",
       "csrc/dense_tc.cuh, dense_tc64.cuh) and `multiple_vs_tc` the shared encoder against",
       "five of those (32x32).", "",
       "## 1-D batches", "", benchmark.report_table(reps, "1d"), "",
       "## 2-D blocks", "", benchmark.report_table(reps, "2d"), "",
       "## absolute throughput (G coefficients / s)", "",
       "| layout | pipeline | size | direction | Gcoef/s | IQR/median |", "|---|---|---|---|---|---|"]
for r in reps:
    out.append(f"| {r.layout} | {r.pipeline} | {r.size} | {r.direction} | "
               f"{r.coefficients_per_second / 1e9:.1f} | {r.dispersion:.3f} |")
text = "\n".join(out) + "\n"
print(text)
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(text)

"""Designer kernel on one band-6 design (N from argv, default 32), a few sweeps
(ncu / timing).  Usage: python tools/prof_designer.py [n] [sweeps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2505_23618_b200 import designer as G  # noqa: E402
from paper_2505_23618_b200.design import Side, SparsityPattern, pattern_schedule_template  # noqa: E402
from paper_2505_23618_b200.transforms import TransformKind, build_transform  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
tmpl = pattern_schedule_template(SparsityPattern.band(6, n))
b = build_transform(TransformKind.DST3, n).entries
d = build_transform(TransformKind.DST7, n).entries
starts = np.stack([G.restart_angles(tmpl.n_rotations, 0, r) for r in range(5)])
G.coordinate_descent(b, d, tmpl, Side.PRE, G.default_alpha(n), starts, 1, 1e-30)  # warm
t0 = time.perf_counter()
runs = G.coordinate_descent(b, d, tmpl, Side.PRE, G.default_alpha(n), starts, sweeps, 1e-30)
dt = time.perf_counter() - t0
print(f"n={n}: {sweeps} sweeps x {tmpl.n_rotations} angles in {dt * 1e3:.1f} ms = "
      f"{dt / sweeps / tmpl.n_rotations * 1e6:.2f} us per angle step")

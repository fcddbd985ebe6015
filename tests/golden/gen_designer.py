"""Golden vectors for the GPU designer, produced by running the REFERENCE's own
coordinate descent (fixture infrastructure; build container only).

    cp -r /root/reference/pkg /tmp/refbuild && (cd /tmp/refbuild && python3 setup.py build_ext --inplace)
    REFPKG=/tmp/refbuild/src python tests/golden/gen_designer.py

For each case: the per-restart objective traces and final angles of
_CoordinateDescent.run (reference design.py:377-543) from the restart angles
optimize_adjustment uses (design.py:546-550), and optimize_adjustment's record
(objective, angles, restart index) -- short runs (a few sweeps), where
floating-point reduction order cannot move the descent far.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REFPKG = os.environ.get("REFPKG", "/tmp/refbuild/src")
sys.path.insert(0, REFPKG)

from dctadjust import design as D  # noqa: E402
from dctadjust.transforms import TransformKind, build_transform  # noqa: E402

CASES = [  # name, n, pattern, side, base, sweeps, restarts
    ("band4_pre_n16", 16, D.SparsityPattern.band(4, 16), D.Side.PRE, TransformKind.DST3, 6, 2),
    ("band6_pre_n32", 32, D.SparsityPattern.band(6, 32), D.Side.PRE, TransformKind.DST3, 3, 1),
    ("sub8_post_n16", 16, D.SparsityPattern.subblock(8, 16), D.Side.POST, TransformKind.DCT2, 6, 2),
    ("sub8_post_n64", 64, D.SparsityPattern.subblock(8, 64), D.Side.POST, TransformKind.DCT2, 3, 1),
]

out: dict[str, np.ndarray] = {}
for name, n, pat, side, base, sweeps, restarts in CASES:
    b = build_transform(base, n)
    d = build_transform(TransformKind.DST7, n)
    cfg = D.DesignConfig(max_iterations=sweeps, restarts=restarts)
    alpha = cfg.resolve_alpha(n)
    tmpl = D.pattern_schedule_template(pat)
    cd = D._CoordinateDescent(b.entries, d.entries, tmpl, side, alpha)
    for r in range(restarts + 1):
        th0 = D._restart_angles(tmpl.n_rotations, cfg.rng_seed, r)
        theta, trace, conv = cd.run(th0, cfg.max_iterations, cfg.tolerance)
        out[f"{name}/r{r}/theta0"] = th0
        out[f"{name}/r{r}/theta"] = theta
        out[f"{name}/r{r}/trace"] = np.array(trace)
    adj = D.optimize_adjustment(b, d, pat, side, cfg)
    out[f"{name}/objective"] = np.array(adj.objective)
    out[f"{name}/angles"] = adj.schedule.angles()
    out[f"{name}/restart"] = np.array(adj.restart_index)
    print(name, adj.objective, adj.restart_index, len(out[f"{name}/r0/trace"]))
np.savez_compressed(Path(__file__).resolve().parent / "designer.npz", **out)

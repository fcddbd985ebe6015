"""Generate the designed-adjustment fixtures with the REFERENCE designer.

Test/fixture infrastructure only: this script imports the reference package
(`dctadjust`, built from /root/reference/pkg into a writable copy) and runs its
own `optimize_adjustment(..., DesignConfig())` (reference design.py:560-613,
seed 0, 4 restarts, 2000 sweeps), then writes each result in the reference's
adjustment text format (`matio.write_adjustment`, matio.py:93-107).  The DCT-8
post designs are derived with `dct8_adjustment_from_dst7` (design.py:677-715).

Usage (in the build container, never on the GPU box):
    cp -r /root/reference/pkg /tmp/refbuild && (cd /tmp/refbuild && python3 setup.py build_ext --inplace)
    REFPKG=/tmp/refbuild/src python tests/golden/gen_adjustments.py [name ...]

Outputs: paper_2505_23618_b200/adjustments/<name>.adj and SHA256SUMS.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

REFPKG = os.environ.get("REFPKG", "/tmp/refbuild/src")
sys.path.insert(0, REFPKG)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

OUT = Path(__file__).resolve().parents[2] / "paper_2505_23618_b200" / "adjustments"

# name -> (pattern label, side, base, target, N)
DESIGNS = {}
for _n in (16, 32, 64):
    DESIGNS[f"band6_pre_dst3_dst7_n{_n}"] = ("band:6", "pre", "dst3", "dst7", _n)
    DESIGNS[f"band4_pre_dst3_dst7_n{_n}"] = ("band:4", "pre", "dst3", "dst7", _n)
    DESIGNS[f"sub8_post_dct2_dst7_n{_n}"] = ("subblock:8", "post", "dct2", "dst7", _n)


def _design(name: str) -> tuple[str, float, str]:
    from dctadjust import matio
    from dctadjust.design import (DesignConfig, Side, SparsityPattern,
                                  optimize_adjustment)
    from dctadjust.transforms import TransformKind, build_transform
    label, side, base, target, n = DESIGNS[name]
    t0 = time.perf_counter()
    adj = optimize_adjustment(
        build_transform(TransformKind(base), n),
        build_transform(TransformKind(target), n),
        SparsityPattern.from_label(label, n),
        Side(side),
        DesignConfig(),
    )
    matio.write_adjustment(OUT / f"{name}.adj", adj)
    info = (f"objective={adj.objective:.6e} identity={adj.identity_objective:.6e} "
            f"converged={adj.converged} restart={adj.restart_index}")
    return name, time.perf_counter() - t0, info


def _derive_dct8() -> None:
    from dctadjust import matio
    from dctadjust.design import dct8_adjustment_from_dst7
    for n in (16, 32, 64):
        src = OUT / f"sub8_post_dct2_dst7_n{n}.adj"
        if src.exists():
            adj = dct8_adjustment_from_dst7(matio.read_adjustment(src))
            matio.write_adjustment(OUT / f"sub8_post_dct2_dct8_n{n}.adj", adj)


def main(argv: list[str]) -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    names = argv or sorted(DESIGNS, key=lambda k: -DESIGNS[k][4])
    with ProcessPoolExecutor(max_workers=min(8, len(names))) as pool:
        for name, dt, info in pool.map(_design, names):
            print(f"{name}: {dt:.1f}s {info}", flush=True)
    _derive_dct8()
    lines = []
    for p in sorted(OUT.glob("*.adj")):
        lines.append(f"{hashlib.sha256(p.read_bytes()).hexdigest()}  {p.name}")
    (OUT / "SHA256SUMS").write_text("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:])

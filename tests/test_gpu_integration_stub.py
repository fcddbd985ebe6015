"""The reference-side binding shown in INTEGRATION.md, executed verbatim: the
backend stub (section 1) against the golden vectors of the seven primitives,
and the fused-entry Axis helper (section 2) against this package's own call."""
import ctypes
import os
import re
import types
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import rel_err  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2505_23618_b200" / "libdctadj.so"


def _blocks():
    text = (ROOT / "INTEGRATION.md").read_text()
    return re.findall(r"```python\n(.*?)```", text, flags=re.S)


def _stub_module():
    os.environ["DCTADJ_LIB"] = str(LIB)
    mod = types.ModuleType("dctadjust_kernels_b200")
    exec(compile(_blocks()[0], "INTEGRATION.md#stub", "exec"), mod.__dict__)
    return mod


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
def test_stub_primitives_match_golden(golden, n):
    b = _stub_module()
    assert b.BACKEND_NAME == "b200"
    x = golden[f"prim/x/{n}"]
    for fn in ("dct2", "idct2", "dst3", "idst3"):
        assert rel_err(getattr(b, fn)(x), golden[f"prim/{fn}/{n}"]) < 1e-9
    for taps in (3, 4, 6):
        if f"prim/band/{n}/{taps}" in golden:
            got = b.band(golden[f"prim/band_a/{n}/{taps}"], taps, x)
            assert rel_err(got, golden[f"prim/band/{n}/{taps}"]) < 1e-9
    for order in (5, 8):
        if f"prim/sub/{n}/{order}" in golden:
            got = b.subblock(golden[f"prim/sub_blk/{n}/{order}"], x)
            assert rel_err(got, golden[f"prim/sub/{n}/{order}"]) < 1e-9
    assert rel_err(b.dense(golden[f"prim/dense_m/{n}"], x), golden[f"prim/dense/{n}"]) < 1e-9


def test_stub_axis_helper_runs_the_fused_entry():
    from paper_2505_23618_b200 import _lib, matio, pipeline
    ns = {"ctypes": ctypes, "np": np, "_DP": ctypes.POINTER(ctypes.c_double)}
    block = next(b for b in _blocks() if "class Axis" in b)
    exec(compile(block, "INTEGRATION.md#axis", "exec"), ns)
    for name in ("band6_pre_dst3_dst7_n32", "sub8_post_dct2_dst7_n32"):
        t = pipeline.make_adjusted_transform(matio.load_designed(name))
        ax, keep = ns["axis"](t)
        x = torch.randn(1000, 32, device="cuda", dtype=torch.float64)
        y = torch.empty_like(x)
        lib = ctypes.CDLL(str(LIB))
        rc = lib.dctadj_forward_1d(ctypes.byref(ax), ctypes.c_void_p(x.data_ptr()),
                                   ctypes.c_void_p(y.data_ptr()), ctypes.c_int64(1000),
                                   ctypes.c_int32(_lib.F64),
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0
        want = pipeline.forward_adjusted(t, x)
        assert rel_err(y.cpu().numpy(), want.cpu().numpy()) < 1e-12

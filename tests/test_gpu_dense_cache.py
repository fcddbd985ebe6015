"""The device cache of dense matrices (csrc/abi.cu upload_dense): entries are
pinned from lookup to launch, evicted least-recently-used, and freed only after
the kernels that read them.  Driven past its 64 slots with calls whose two axes
upload two different matrices (the case where FIFO eviction used to free the
first upload of the same call before its kernel ran)."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import rel_err  # noqa: E402

pytestmark = pytest.mark.gpu


def _state():
    from paper_2505_23618_b200 import _lib
    e, p = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.load().dctadj_dense_cache_state(ctypes.byref(e), ctypes.byref(p)))
    return e.value, p.value


def _dense_t(m):
    from paper_2505_23618_b200 import pipeline
    from paper_2505_23618_b200.design import (AdjustmentMatrix, Side, SparsityPattern,
                                              pattern_schedule_template)
    from paper_2505_23618_b200.transforms import TransformKind
    n = m.shape[0]
    pat = SparsityPattern.dense(n)
    adj = AdjustmentMatrix(pat, Side.POST, TransformKind.DCT2, TransformKind.DST7,
                           pattern_schedule_template(pat), m)
    return pipeline.make_adjusted_transform(adj)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_cache_overflow_keeps_results(dtype):
    from paper_2505_23618_b200 import kernels, pipeline
    from paper_2505_23618_b200.transforms import TransformKind, build_transform
    rng = np.random.default_rng(5)
    d2 = build_transform(TransformKind.DCT2, 32).entries
    x = torch.from_numpy(rng.standard_normal((64, 32, 32))).to("cuda", dtype)
    xv = torch.from_numpy(rng.standard_normal((97, 32))).to("cuda", dtype)
    tol = 1e-5 if dtype == torch.float32 else 1e-9
    for i in range(90):  # > 64 slots: every 2-D call evicts while uploading its second axis
        q_h, _ = np.linalg.qr(rng.standard_normal((32, 32)))
        q_v, _ = np.linalg.qr(rng.standard_normal((32, 32)))
        m = rng.standard_normal((32, 32))
        yv = kernels.dense(m, xv)  # one more distinct entry per iteration
        th, tv = _dense_t(q_h @ d2.T), _dense_t(q_v @ d2.T)
        y = pipeline.forward_adjusted_2d(th, tv, x)
        if i % 15 == 0 or i > 80:
            ref = np.einsum("ri,bij,cj->brc", q_v, x.double().cpu().numpy(), q_h)
            assert rel_err(y.cpu().numpy(), ref) < tol, i
            assert rel_err(yv.cpu().numpy(), xv.double().cpu().numpy() @ m.T) < tol, i
        entries, pinned = _state()
        assert pinned == 0, (i, entries, pinned)  # every call unpins what it used
        assert entries <= 64 + 2

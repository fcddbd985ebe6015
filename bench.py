"""Benchmark: transform coefficients/s (forward + inverse each counted) of the
adjusted-transform hot path on B200, with the roofline and the reference CPU
path beside it.

    python bench.py [--gpus N --steps K --warmup W] [--config c2] [--impl ours|reference]

Default workload (BASELINE.json configs[1], the config the metric is quoted on
that fits one GPU): 65,536 blocks of 32x32 fp32 integer residuals (AR(1)
rho=0.85, sigma=24, clipped to [-512, 511]), forward + inverse DCT-8
approximation = DCT-2 butterfly + designed 8x8 post-adjustment on both axes.
One step = forward_adjusted_2d then inverse_adjusted_2d over the batch, each one
fused kernel (rows + columns + adjustment).  Inputs are 268 MB per GPU (> the
126 MB L2), so no flush is needed between steps.

The other configs (--config c1 | c3_pre | c3_post | c4_{dst7,dct8}_{pre,post} |
c5) are parity cases of BASELINE.json measured the same way (no bench line).

Multi-GPU (torchrun): every rank runs the same per-GPU workload on its own
block range (weak scaling, no data-path collective); timing is CUDA events on
the launching stream, max over ranks (NCCL all_reduce of scalars only).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "transform coeffs/sec (fwd+inv) at 1/2/4/8 B200; % of HBM roofline vs CPU ref"
UNIT = "coef/s"


# ------------------------------------------------------------------ adjustments
def _t(adj):
    from paper_2505_23618_b200 import pipeline
    return pipeline.make_adjusted_transform(adj)


def _post(n, kind):
    from paper_2505_23618_b200 import matio
    from paper_2505_23618_b200.design import dct8_adjustment_from_dst7
    a = matio.load_designed(f"sub8_post_dct2_dst7_n{n}")
    return _t(a if kind == "dst7" else dct8_adjustment_from_dst7(a))


def _pre(n, kind):
    from paper_2505_23618_b200 import matio
    from paper_2505_23618_b200.design import flip_pre_adjustment
    a = matio.load_designed(f"band6_pre_dst3_dst7_n{n}")
    return _t(a if kind == "dst7" else flip_pre_adjustment(a))


def _oaxis(t):
    from oracle import oracle as O
    adj = t.adjustment
    base = {"dct2": O.BASE_DCT2, "dst3": O.BASE_DST3, "dct3": O.BASE_DCT3}[adj.base.value]
    kind = {"band": O.ADJ_BAND, "subblock": O.ADJ_SUBBLOCK, "dense": O.ADJ_DENSE}[adj.pattern.kind.value]
    return O.OAxis(adj.pattern.size, base, kind, O.SIDE_PRE if adj.side.value == "pre" else O.SIDE_POST,
                   adj.pattern.taps or 0, adj.pattern.order or 0, np.array(adj.realized))


# uniform-block configs: (workload, blocks, H=W, dtype, transform factory, inputs, inverse?)
UNIFORM = {
    "c2": ("c2_dct8_post_sub8_n32_fwd+inv_65536x32x32", 65536, 32, "f32",
           lambda: _post(32, "dct8"), "c2_inputs", True),
    "c1": ("c1_dst7_pre_band6_n32_fwd_4096x32x32", 4096, 32, "f64",
           lambda: _pre(32, "dst7"), "c1_inputs", False),
}
for _k in ("dst7", "dct8"):
    UNIFORM[f"c4_{_k}_pre"] = (f"c4_{_k}_pre_band6_n64_fwd+inv_262144x64x64", 262144, 64, "f32",
                               (lambda k=_k: _pre(64, k)), "c4_inputs", True)
    UNIFORM[f"c4_{_k}_post"] = (f"c4_{_k}_post_sub8_n64_fwd+inv_262144x64x64", 262144, 64, "f32",
                                (lambda k=_k: _post(64, k)), "c4_inputs", True)
CONFIGS = sorted(UNIFORM) + ["c3_pre", "c3_post", "c5"]


# ------------------------------------------------------------------ helpers
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms by one
    long-running `nvidia-smi -lms 50`; only samples that arrive inside the
    timed window (mark_start .. mark_end) are summarised."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []  # (arrival time, fields)
        self.t0 = self.t1 = None
        self._proc = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            for line in self._proc.stdout:
                if line.strip():
                    self.samples.append((time.time(), [x.strip() for x in line.split(",")]))
        except Exception:
            pass

    def __enter__(self):
        self._t.start()
        time.sleep(0.3)  # let nvidia-smi start before the timed region
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *exc):
        time.sleep(0.1)
        if self._proc is not None:
            self._proc.terminate()
        self._t.join(timeout=5)

    def summary(self):
        win = [f for (t, f) in self.samples
               if self.t0 is not None and self.t1 is not None and self.t0 - 0.05 <= t <= self.t1 + 0.05]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        num = lambda v: v.replace(".", "", 1).isdigit()  # noqa: E731
        sm = [float(f[0]) for f in win if num(f[0])]
        mx = [float(f[1]) for f in win if num(f[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for f in win for i in range(4)
                          if len(f) > 2 + i and f[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(win)}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _traffic(workload: str, launch: str):
    """ncu dram bytes (read + write) of one `launch` of `workload`, from
    profiles/ncu_traffic.json (keys "<workload>/<launch>")."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        return json.loads(p.read_text()).get(f"{workload}/{launch}")
    return None


def _block_err(got: np.ndarray, ref: np.ndarray) -> float:
    n = got.shape[0]
    num = np.abs(got.astype(np.float64) - ref).reshape(n, -1).max(1)
    den = np.maximum(np.abs(ref).reshape(n, -1).max(1), 1e-300)
    return float((num / den).max())


# ------------------------------------------------------------------ GPU workloads
class Workload:
    """One config on one rank: device buffers, the launches of one step, the
    oracle gate, and (uniform configs) the host-buffer e2e step."""

    workload = ""
    dtype = "f32"
    launches: list = []          # [(name, callable)] per step, in order
    coef_per_step = 0            # coefficients produced per step (all transforms)
    bytes_first_launch = 0       # algorithmic bytes of launches[0]
    e2e = None                   # callable for one end-to-end step, or None
    e2e_bytes = (0, 0)
    e2e_api = ""
    extra: dict = {}
    kernels_per_step = None      # device kernels launched per step (default: one per launch)
    kernel_name = "tile_kernel"  # the library kernel behind launches[0]

    def gate(self) -> float:
        raise NotImplementedError

    def check_e2e(self):
        pass


class Uniform(Workload):
    def __init__(self, name: str, rank: int, fused_roundtrip: bool = False):
        import torch
        from paper_2505_23618_b200 import _lib, pipeline, workloads
        wl, nblk, n, dt, make, inputs, inverse = UNIFORM[name]
        self.workload, self.dtype = wl, dt
        self.t = make()
        self.nblk = nblk
        self.x = getattr(workloads, inputs)("cuda", nblk, offset=rank * nblk)
        self.y = torch.empty_like(self.x)
        self.xr = torch.empty_like(self.x)
        coef = nblk * n * n
        es = self.x.element_size()
        self.inverse = inverse
        self.coef_per_step = coef * (2 if inverse else 1)
        self.bytes_first_launch = 2 * coef * es
        lib = _lib.load()
        ax, self._keep = self.t.axis()
        self.ax = ax
        dtc = _lib.F32 if dt == "f32" else _lib.F64
        st = torch.cuda.current_stream().cuda_stream
        ref = ctypes.byref(ax)

        def fwd():
            _lib.check(lib.dctadj_forward_2d(ref, ref, self.x.data_ptr(), self.y.data_ptr(), nblk, dtc, st))

        def inv():
            _lib.check(lib.dctadj_inverse_2d(ref, ref, self.y.data_ptr(), self.xr.data_ptr(), nblk, dtc, st))

        def rt():  # forward + inverse in one kernel: x read once, y and x' written once
            _lib.check(lib.dctadj_roundtrip_2d(ref, ref, self.x.data_ptr(), self.y.data_ptr(),
                                               self.xr.data_ptr(), nblk, dtc, st))

        self.two_kernel = [("forward_2d", fwd)] + ([("inverse_2d", inv)] if inverse else [])
        self.launches = self.two_kernel
        if fused_roundtrip and inverse and lib.dctadj_roundtrip_fused(ref, ref, dtc):
            self.launches = [("roundtrip_2d", rt)]
            self.bytes_first_launch = 3 * coef * es
            self.kernel_name = "roundtrip_kernel"
        self._lib, self._dtc, self._st, self._ref = lib, dtc, st, ref
        # e2e: the same step through the host-buffer entries (pinned arrays)
        self.xh = self.x.cpu().pin_memory().numpy()
        self.yh = torch.empty(tuple(self.x.shape), dtype=self.x.dtype).pin_memory().numpy()
        self.xrh = torch.empty(tuple(self.x.shape), dtype=self.x.dtype).pin_memory().numpy()

        def e2e():
            if inverse:  # the round trip in one pipelined pass (coefficients D2H once)
                pipeline.roundtrip_adjusted_2d_host(self.t, self.t, self.xh, out=self.yh,
                                                    out_inv=self.xrh)
            else:
                pipeline.forward_adjusted_2d_host(self.t, self.t, self.xh, out=self.yh)

        self.e2e = e2e
        nb = coef * es
        # round trip: x in once; coefficients and reconstruction out
        self.e2e_bytes = (nb, nb * (2 if inverse else 1))
        self.e2e_api = ("roundtrip_adjusted_2d_host (C-ABI dctadj_roundtrip_2d_host)" if inverse
                        else "forward_adjusted_2d_host (C-ABI dctadj_forward_2d_host)")
        self.extra = {"blocks_per_gpu": nblk, "block": f"{n}x{n}",
                      "l2": f"inputs {nb / 1e6:.0f} MB per GPU "
                            + ("> 126 MB L2; no flush" if nb > 126e6 else "< 126 MB L2: L2-resident")}

    def rotating(self, min_bytes: float = 1.0e9):
        """L2-resident configs (C1): step functions over R distinct input/output
        buffer pairs, R chosen so one cycle moves >= min_bytes (8x the 126 MB L2);
        the survey asks for this number beside the resident one."""
        import torch
        from paper_2505_23618_b200 import _lib
        nb = self.x.numel() * self.x.element_size()
        r = max(2, int(np.ceil(min_bytes / (2 * nb))))
        xs = [self.x.clone() for _ in range(r)]
        ys = [torch.empty_like(self.x) for _ in range(r)]
        lib, dtc, st, ref, nblk = self._lib, self._dtc, self._st, self._ref, self.nblk

        def step(i):
            _lib.check(lib.dctadj_forward_2d(ref, ref, xs[i].data_ptr(), ys[i].data_ptr(), nblk, dtc, st))
            if self.inverse:
                _lib.check(lib.dctadj_inverse_2d(ref, ref, ys[i].data_ptr(), xs[i].data_ptr(), nblk,
                                                 dtc, st))
        return r, step

    def gate(self):
        import torch
        from oracle import oracle as O
        from paper_2505_23618_b200 import pipeline
        y0 = pipeline.forward_adjusted_2d(self.t, self.t, self.x)
        idx = torch.arange(0, self.nblk, max(1, self.nblk // 256), device="cuda")
        xs = self.x[idx].cpu().numpy().astype(np.float64)
        ax = _oaxis(self.t)
        return _block_err(y0[idx].cpu().numpy(), O.adjusted_2d(ax, ax, xs))

    def check_e2e(self):
        import torch
        torch.cuda.synchronize()
        if not np.array_equal(self.yh, self.y.cpu().numpy()):
            raise SystemExit("e2e coefficients differ from the device path")
        if self.inverse and self.workload.startswith("c2"):
            if not np.array_equal(np.rint(self.xrh), self.xh):
                raise SystemExit("e2e round trip lost integer exactness")


class Mixed(Workload):
    """Config 3: 1,048,576 blocks, shapes {16,32}^2 and (h, v) kinds uniform."""

    def __init__(self, side: str, rank: int, nblk: int = 1 << 20, fused_roundtrip: bool = False):
        import torch
        from paper_2505_23618_b200 import _lib, pipeline, workloads
        self.workload = f"c3_mixed_{side}_fwd+inv_{nblk}blocks"
        g_h, g_w, kinds = workloads.c3_shapes(nblk, seed=3 + 1000 * rank)
        h_kind, v_kind = (kinds % 2).numpy(), (kinds // 2).numpy()
        sizes = np.array([16, 16, 32, 32])
        h_index = (np.where(g_w.numpy() == 16, 0, 2) + h_kind).astype(np.int32)
        v_index = (np.where(g_h.numpy() == 16, 0, 2) + v_kind).astype(np.int32)
        self.batch = pipeline.MixedBatch.packed(h_index, v_index, sizes)
        if side == "pre":
            self.table = [_pre(16, "dst7"), _pre(16, "dct8"), _pre(32, "dst7"), _pre(32, "dct8")]
        else:
            self.table = [_post(16, "dst7"), _post(16, "dct8"), _post(32, "dst7"), _post(32, "dct8")]
        # inputs: Laplace-innovation AR(1) blocks, generated per shape and scattered
        total = self.batch.total_elements
        self.x = torch.empty(total, device="cuda", dtype=torch.float32)
        offs = torch.from_numpy(self.batch.offsets).cuda()
        hh = torch.from_numpy(sizes[v_index]).cuda()
        ww = torch.from_numpy(sizes[h_index]).cuda()
        for si, (H, W) in enumerate(((16, 16), (16, 32), (32, 16), (32, 32))):
            sel = torch.nonzero((hh == H) & (ww == W)).flatten()
            if sel.numel() == 0:
                continue
            blocks = workloads.c3_block(H, W, sel.numel(), seed=3 * 1_000_003 + 97 * rank + si)
            idx = offs[sel][:, None] + torch.arange(H * W, device="cuda")[None, :]
            self.x[idx.flatten()] = blocks.reshape(-1)
            del blocks, idx
        self.y = torch.empty_like(self.x)
        self.xr = torch.empty_like(self.x)
        self.coef_per_step = 2 * total
        self.bytes_first_launch = 2 * total * 4
        self.axes = (_lib.Axis * 4)()
        self._keep = []
        for k, tr in enumerate(self.table):
            ax, m = tr.axis()
            self.axes[k] = ax
            self._keep.append(m)
        lib = _lib.load()
        st = torch.cuda.current_stream().cuda_stream
        plan = self.batch._plan

        def fwd():
            _lib.check(lib.dctadj_mixed_forward(plan, self.axes, self.x.data_ptr(), self.y.data_ptr(), 0, st))

        def inv():
            _lib.check(lib.dctadj_mixed_inverse(plan, self.axes, self.y.data_ptr(), self.xr.data_ptr(), 0, st))

        def rt():  # one fused gather kernel per class: x read once, y and x' written once
            _lib.check(lib.dctadj_mixed_roundtrip(plan, self.axes, self.x.data_ptr(), self.y.data_ptr(),
                                                  self.xr.data_ptr(), 0, st))

        self.two_kernel = [("mixed_forward", fwd), ("mixed_inverse", inv)]
        self.launches = self.two_kernel
        nclass = len(self.batch_classes(h_index, v_index))
        self.kernels_per_step = 2 * nclass
        if fused_roundtrip and lib.dctadj_mixed_roundtrip_fused(plan, self.axes, 0):
            self.launches = [("mixed_roundtrip", rt)]
            self.kernels_per_step = nclass
            self.bytes_first_launch = 3 * total * 4
            self.kernel_name = "roundtrip_kernel (gather, one per class)"
        self.h_index, self.v_index = h_index, v_index
        self.extra = {"blocks_per_gpu": nblk, "coefficients_per_gpu": total,
                      "classes": int(len(np.unique(h_index * 4 + v_index))),
                      "l2": f"inputs {total * 4 / 1e6:.0f} MB per GPU > 126 MB L2; no flush"}

    @staticmethod
    def batch_classes(h_index, v_index):
        return np.unique(np.asarray(h_index) * 4 + np.asarray(v_index))

    def gate(self):
        from oracle import oracle as O
        from paper_2505_23618_b200 import pipeline
        y = pipeline.mixed_forward(self.batch, self.table, self.x).cpu().numpy()
        x = self.x.cpu().numpy()
        worst = 0.0
        for i in range(0, self.batch.nblk, max(1, self.batch.nblk // 256)):
            o = int(self.batch.offsets[i])
            h, w = int(self.batch.sizes[self.v_index[i]]), int(self.batch.sizes[self.h_index[i]])
            ref = O.adjusted_2d(_oaxis(self.table[self.h_index[i]]), _oaxis(self.table[self.v_index[i]]),
                                x[o:o + h * w].reshape(1, h, w).astype(np.float64))
            worst = max(worst, _block_err(y[o:o + h * w].reshape(1, h, w), ref))
        return worst


class Frames(Workload):
    """Config 5: 64 frames 3840x2160 fp32 per GPU, 32x32 tiles (bottom padded to
    2176 rows by TMA zero fill); adjusted DST-7 (sub8 post) forward + inverse
    plus the exact dense DST-7 forward on the same tiles.  The coefficient-
    domain approximation error sum|Y_adj - Y_exact|^2 / sum|Y_exact|^2 is
    reported over all tiles and over the 67 unpadded tile rows."""

    def __init__(self, rank: int, world: int, nframes: int = 64):
        import torch
        from paper_2505_23618_b200 import _lib, pipeline, shard, workloads
        from paper_2505_23618_b200.design import (AdjustmentMatrix, Side, SparsityPattern,
                                                  pattern_schedule_template)
        from paper_2505_23618_b200.transforms import TransformKind, build_transform
        f0, f1 = shard.frame_range(rank, world, nframes * world)  # weak scaling: 64 per GPU
        self.nframes = f1 - f0
        self.H, self.W = 2160, 3840
        self.workload = f"c5_frames_{self.nframes}x3840x2160_dst7_post_sub8_fwd+inv+dense_exact"
        self.frames = workloads.c5_frames(self.nframes, self.H, self.W, offset=f0)
        self.t = _post(32, "dst7")
        d7 = build_transform(TransformKind.DST7, 32).entries
        c = d7 @ build_transform(TransformKind.DCT2, 32).entries.T
        dense = AdjustmentMatrix(SparsityPattern.dense(32), Side.POST, TransformKind.DCT2,
                                 TransformKind.DST7, pattern_schedule_template(SparsityPattern.dense(32)), c)
        self.td = pipeline.make_adjusted_transform(dense)
        nblk = pipeline.frame_block_count(self.nframes, self.H, self.W, 32, 32)
        self.y = torch.empty(nblk, 32, 32, device="cuda")
        self.ye = torch.empty_like(self.y)
        self.back = torch.empty_like(self.frames)
        lib = _lib.load()
        st = torch.cuda.current_stream().cuda_stream
        (ax, k1), (axd, k2) = self.t.axis(), self.td.axis()
        self._keep = (ax, k1, axd, k2)
        r, rd = ctypes.byref(ax), ctypes.byref(axd)
        F, H, W = self.nframes, self.H, self.W

        def fwd():
            _lib.check(lib.dctadj_forward_frames(r, r, self.frames.data_ptr(), self.y.data_ptr(), F, H, W, 0, st))

        def inv():
            _lib.check(lib.dctadj_inverse_frames(r, r, self.y.data_ptr(), self.back.data_ptr(), F, H, W, 0, st))

        self.err = torch.zeros((F, 4), dtype=torch.float64, device="cuda")

        def fwd_exact():  # adjusted + exact forward and the error sums, one read of the frames
            _lib.check(lib.dctadj_forward_frames_exact(r, r, rd, rd, self.frames.data_ptr(),
                                                       self.y.data_ptr(), self.ye.data_ptr(),
                                                       self.err.data_ptr(), F, H, W, 0, st))

        self.launches = [("forward_frames_exact", fwd_exact), ("inverse_frames", inv)]
        self.kernel_name = "dense_tc_kernel<FRAME4, FUSED sub8-post>"
        # the same three transforms as separate kernels (error sums not included)
        self.two_kernel = [("forward_frames", fwd), ("dense_dst7_frames",
                           lambda: _lib.check(lib.dctadj_forward_frames(
                               rd, rd, self.frames.data_ptr(), self.ye.data_ptr(), F, H, W, 0, st))),
                           ("inverse_frames", inv)]
        coef = nblk * 1024
        self.coef_per_step = 3 * coef
        self.bytes_first_launch = 4 * (F * H * W + 2 * coef)
        self.extra = {"frames_per_gpu": F, "blocks_per_gpu": nblk, "padded_rows": 2176,
                      "coefficients_padded": coef, "coefficients_unpadded": F * H * W,
                      "step": "fused [adjusted DST-7 forward + exact dense DST-7 forward + per-frame "
                              "error sums] (one read of the frames) + adjusted inverse; value counts "
                              "all three transforms"}

    def gate(self):
        from oracle import oracle as O
        from paper_2505_23618_b200 import pipeline
        y = pipeline.forward_frames(self.t, self.t, self.frames[:1])
        pad = np.zeros((2176, 3840))
        pad[:2160] = self.frames[0].cpu().numpy()
        blocks = pad.reshape(68, 32, 120, 32).transpose(0, 2, 1, 3).reshape(-1, 32, 32)
        sel = np.arange(0, blocks.shape[0], 37)
        ax = _oaxis(self.t)
        return _block_err(y.cpu().numpy()[sel], O.adjusted_2d(ax, ax, blocks[sel]))

    def approximation_error(self):
        """From the fused launch's own per-frame sums, cross-checked against a
        torch fp64 reduction over its two outputs."""
        e = self.err.sum(dim=0).tolist()
        chk = self._approximation_error_torch()
        if not np.allclose(e, chk, rtol=1e-4):
            raise SystemExit(f"fused error sums {e} disagree with the outputs {chk}")
        return e

    def _approximation_error_torch(self):
        y = self.y.view(self.nframes, 68, 120, 32, 32).double()
        ye = self.ye.view(self.nframes, 68, 120, 32, 32).double()
        d_all = (y - ye).pow(2).sum().item()
        e_all = ye.pow(2).sum().item()
        d_full = (y[:, :67] - ye[:, :67]).pow(2).sum().item()
        e_full = ye[:, :67].pow(2).sum().item()
        return [d_all, e_all, d_full, e_full]


# ------------------------------------------------------------------ CPU legs
def _cpu_worker(args):
    kind, cfg_name, nblk, seed, reps = args
    from oracle import oracle as O
    wl, _, n, _, make, _, inverse = UNIFORM[cfg_name]
    ax = _oaxis(make())
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((nblk, n, n)) * 24.0
    if kind == "reference":
        ref = O.RefPipeline()
        fwd = lambda a: ref.forward_2d(ax, ax, a)  # noqa: E731
        inv = lambda a: ref.inverse_2d(ax, ax, a)  # noqa: E731
    else:
        fwd = lambda a: O.adjusted_2d(ax, ax, a)  # noqa: E731
        inv = lambda a: O.adjusted_2d(ax, ax, a, inverse=True)  # noqa: E731
    t0 = time.perf_counter()
    for _ in range(reps):
        y = fwd(x)
        if inverse:
            inv(y)
    return time.perf_counter() - t0


def cpu_throughput(cfg_name: str, seconds: float = 8.0, pool=None, reps: int = 0):
    """Reference CPU path on this host's cores: the reference's compiled core
    (oracle/_ref, kind "reference") when built, else the C port (kind "port");
    one process per core, each on its own block sample, single-threaded BLAS.
    `reps` > 0 fixes the passes per process (else sized to ~`seconds`); `pool`
    reuses a caller's fork pool."""
    from multiprocessing import get_context
    from oracle import oracle as O
    if cfg_name not in UNIFORM:
        cfg_name = "c2"
    wl, _, n, _, _, _, inverse = UNIFORM[cfg_name]
    kind = "reference" if O.ref_fastcore() is not None else "port"
    cores = O.threads_available()
    nblk = 256 if n == 32 else 64
    per_pass = nblk * n * n * (2 if inverse else 1)
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    if reps <= 0:
        t1 = _cpu_worker((kind, cfg_name, nblk, 0, 1))
        reps = max(1, int(seconds / max(t1, 1e-6)))
    jobs = [(kind, cfg_name, nblk, s, reps) for s in range(cores)]
    if pool is None:
        with get_context("fork").Pool(cores) as own:
            times = own.map(_cpu_worker, jobs)
    else:
        times = pool.map(_cpu_worker, jobs)
    value = cores * reps * per_pass / max(times)
    sample = (f"{cores} processes x {reps} passes x {nblk} blocks ({n}x{n}, "
              f"{'fwd+inv' if inverse else 'fwd'}) of the {cfg_name} workload")
    return {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}


def run_reference(args, rank: int, world: int):
    """`--impl reference`: the reference's CPU path alone (rank 0; other ranks exit).
    Each step is a bounded sample of the workload on every host core; the sample
    is sized so the whole --warmup + --steps run takes about `--ref-seconds`."""
    if rank != 0:
        return
    from multiprocessing import get_context
    from oracle import oracle as O
    cfg = args.config if args.config in UNIFORM else "c2"
    wl, _, n, dt, _, _, _ = UNIFORM[cfg]
    nsteps = args.warmup + args.steps
    per_step = min(2.0, max(0.02, args.ref_seconds / nsteps))
    kind = "reference" if O.ref_fastcore() is not None else "port"
    nblk = 256 if n == 32 else 64
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    t1 = _cpu_worker((kind, cfg, nblk, 0, 1))
    reps = max(1, int(per_step / max(t1, 1e-6)))
    per = []
    res = None
    with get_context("fork").Pool(O.threads_available()) as pool:
        for i in range(nsteps):
            r = cpu_throughput(cfg, pool=pool, reps=reps)
            if i >= args.warmup:
                per.append(r["value"])
                res = r
    value = float(np.median(per))
    res["value"] = value
    per_step_coefs = O.threads_available() * reps * nblk * n * n * (2 if UNIFORM[cfg][6] else 1)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step_coefs / value * 1e3,
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic",
            "impl": "reference", "config": {"workload": wl, "sample_per_step": res["sample"]},
            "cpu_baseline": res,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.config in UNIFORM:
        w = Uniform(args.config, rank, fused_roundtrip=not args.unfused)
    elif args.config.startswith("c3"):
        w = Mixed(args.config.split("_")[1], rank, fused_roundtrip=not args.unfused)
    else:
        w = Frames(rank, world)
    torch.cuda.synchronize()

    # oracle gate before timing (reference benchmark.py:181-190)
    err = w.gate()
    tol = 1e-5 if w.dtype == "f32" else 1e-9
    if err > tol:
        raise SystemExit(f"oracle gate failed: rel err {err:.3e} > {tol}")

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        for _, fn in w.launches:
            fn()
    torch.cuda.synchronize()
    # every output of a warm-up step is finite (the oracle gate samples blocks)
    for name in ("y", "xr", "ye", "back"):
        t = getattr(w, name, None)
        if t is not None and not bool(torch.isfinite(t).all()):
            raise SystemExit(f"non-finite values in {name} after the warm-up steps")

    # timed region: K steps back to back, CUDA events only at its two ends (an
    # event between launches would serialise the kernels' programmatic launch)
    nl = len(w.launches)
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark_start()
        e_start.record(stream)
        for _ in range(args.steps):
            for _, fn in w.launches:
                fn()
        e_end.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
        if world > 1:
            dist.barrier()
    total_ms = e_start.elapsed_time(e_end)
    # per-kernel durations (roofline): each launch type back to back on the
    # same stream, CUDA events around the run
    per_launch_ms = []
    reps = max(10, min(args.steps, 200))
    for _, fn in w.launches:
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        per_launch_ms.append(a.elapsed_time(b) / reps)

    unfused = None  # fused round trips: the same step as forward + inverse kernels, for reference
    if getattr(w, "two_kernel", None) is not None and w.two_kernel is not w.launches:
        ums = []
        for _, fn in w.two_kernel:
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            ums.append(a.elapsed_time(b) / reps)
        unfused = {"value": w.coef_per_step / (sum(ums) / 1e3),
                   "per_launch_ms": dict(zip([n for n, _ in w.two_kernel], ums)),
                   "note": "the same transforms as separate kernels, each reading its input "
                           "from HBM (round trips: 16 B per coefficient pair instead of 12)"}

    # dispersion: per-step CUDA events over up to 50 further steps (median, IQR)
    nsamp = min(args.steps, 50)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(nsamp + 1)]
    ev[0].record(stream)
    for i in range(nsamp):
        for _, fn in w.launches:
            fn()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    step_ms = np.array([ev[i].elapsed_time(ev[i + 1]) for i in range(nsamp)])
    q1, med, q3 = np.percentile(step_ms, [25, 50, 75])
    dispersion = {"median_ms_per_step": float(med), "iqr_ms": float(q3 - q1), "samples": nsamp,
                  "note": "per-step events (separate pass after the timed region)"}

    rot = None
    if isinstance(w, Uniform) and w.bytes_first_launch < 126e6:
        nbuf, step = w.rotating()
        for i in range(nbuf):
            step(i)
        torch.cuda.synchronize()
        nrot = max(args.steps, 2 * nbuf)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(nrot):
            step(i % nbuf)
        b.record(stream)
        torch.cuda.synchronize()
        rms = a.elapsed_time(b) / nrot
        rot = {"value": w.coef_per_step / (rms / 1e3), "ms_per_step": rms, "buffers": nbuf,
               "note": "inputs rotate over buffers totalling > 8x L2 (not L2-resident)"}

    e2e_s = None
    if w.e2e is not None:
        w.e2e()  # warm
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2e_steps = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            w.e2e()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        w.check_e2e()

    approx = w.approximation_error() if isinstance(w, Frames) else None

    if world > 1:
        t = torch.tensor([total_ms, e2e_s or 0.0], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_s = float(t[0]), (float(t[1]) if e2e_s is not None else None)
        if approx is not None:
            a = torch.tensor(approx, device="cuda", dtype=torch.float64)
            dist.all_reduce(a, op=dist.ReduceOp.SUM)
            approx = a.tolist()

    ms_per_step = total_ms / args.steps
    value = world * w.coef_per_step / (ms_per_step / 1e3)
    peak, peak_src = _peaks()
    achieved = w.bytes_first_launch / (per_launch_ms[0] / 1e3) / 1e9
    config = {"workload": w.workload, "parallelism": f"block-range shards x{world}",
              "oracle_gate_rel_err": err}
    config.update(w.extra)
    if rot is not None:
        config["l2_rotating_buffers"] = rot
    if unfused is not None:
        config["schedule"] = f"fused: {', '.join(n for n, _ in w.launches)}"
        config["unfused_separate_kernels"] = unfused
    if approx is not None:
        config["approx_error_vs_exact_dst7_all_tiles"] = approx[0] / approx[1]
        config["approx_error_vs_exact_dst7_unpadded_tile_rows"] = approx[2] / approx[3]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": w.dtype,
        "data": "synthetic (seeded residual fields per BASELINE.json configs, SURVEY.md App. A D12)",
        "config": config,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic(w.workload, w.launches[0][0]),
                     "peak_source": peak_src,
                     "kernel": f"{w.kernel_name} ({w.launches[0][0]})",
                     "algorithmic_bytes_per_launch": w.bytes_first_launch,
                     "avg_launch_ms": per_launch_ms[0],
                     "per_launch_ms": dict(zip([n for n, _ in w.launches], per_launch_ms))},
        "e2e": ({"value": world * w.coef_per_step / e2e_s, "unit": UNIT,
                 "h2d_bytes_per_step": w.e2e_bytes[0], "d2h_bytes_per_step": w.e2e_bytes[1],
                 "api": w.e2e_api}
                if e2e_s else None),
        "gpu_launches": args.steps * (w.kernels_per_step or nl),
        "clocks": clk.summary(),
        "dispersion": dispersion,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_throughput(args.config, seconds=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=CONFIGS)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--unfused", action="store_true",
                    help="fwd+inv configs: time forward and inverse as two kernels (x, y each "
                         "cross HBM twice) instead of the fused round trip")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--ref-seconds", type=float, default=120.0,
                    help="--impl reference: total CPU time budget over warmup + steps")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

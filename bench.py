"""Benchmark: transform coefficients/s (forward + inverse each counted) of the
adjusted-transform hot path on B200, with the roofline and the reference CPU
path beside it.

    python bench.py [--gpus N --steps K --warmup W] [--config c2] [--impl ours|reference]
                    [--scaling strong|weak] [--no-per-config] [--dry-run]

Headline (BASELINE.json configs[1], the config the metric is quoted on that fits
one GPU): 65,536 blocks of 32x32 fp32 integer residuals (AR(1) rho=0.85,
sigma=24, clipped to [-512, 511]), forward + inverse DCT-8 approximation =
DCT-2 butterfly + designed 8x8 post-adjustment on both axes; one step = the
fused round-trip kernel over the batch.  The same run measures every other
config of BASELINE.json the same way (`config.per_config`): C1 fp64 band-6 pre
DST-7 forward, C3 mixed shapes pre / post, C4 64x64 x 4 variants, C5 4K frames
with the exact dense DST-7 comparison.

Multi-GPU (reference SPEC.md:313-314: blocks are independent):
`--gpus N` launches N ranks (torchrun, one per GPU) unless it already runs
under one.  Scaling is STRONG by default: the config's total work is split --
C1 / C2 / C4 by contiguous block range (shard.block_range), C3 at equal
coefficient counts (shard.weighted_ranges), C5 by frame (shard.frame_range) --
with no collective on the data path; after timing, NCCL carries scalars only
(shard.reduce_stats: max time, summed counts and error energies, max error).
`--scaling weak` runs the whole config on every rank instead.

Timing: CUDA events on the launching stream around K back-to-back steps, max
over ranks.  Between steps L2 never holds the step's inputs: when a rank's
shard is smaller than the 126 MB L2, the steps rotate over R copies of the
buffers whose bytes exceed 4x L2 (`config.l2`).  Every config is gated against
the CPU oracle over its WHOLE shard (every block, forward and inverse) before
it is timed, as the reference's benchmark.py:181-190 does.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import socket
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
L2_BYTES = 126e6
ROTATE_BYTES = 4 * L2_BYTES   # bytes the rotating buffer sets must cycle through
GATE_CHUNK_BYTES = 256 << 20  # host staging per gate chunk
SETS_OVERRIDE = int(os.environ.get("BENCH_SETS", "0"))  # diagnostics: exactly N buffer sets
INPROC = os.environ.get("BENCH_INPROC", "0") == "1"  # diagnostics: per_config in this process


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


# uniform-block configs: (label, total blocks, H=W, dtype, transform factory, inputs, inverse?)
UNIFORM = {
    "c2": ("c2_dct8_post_sub8_n32_fwd+inv", 65536, 32, "f32", lambda: _post(32, "dct8"), "c2_inputs", True),
    "c1": ("c1_dst7_pre_band6_n32_fwd", 4096, 32, "f64", lambda: _pre(32, "dst7"), "c1_inputs", False),
}
for _k in ("dst7", "dct8"):
    UNIFORM[f"c4_{_k}_pre"] = (f"c4_{_k}_pre_band6_n64_fwd+inv", 262144, 64, "f32",
                               (lambda k=_k: _pre(64, k)), "c4_inputs", True)
    UNIFORM[f"c4_{_k}_post"] = (f"c4_{_k}_post_sub8_n64_fwd+inv", 262144, 64, "f32",
                                (lambda k=_k: _post(64, k)), "c4_inputs", True)
CONFIGS = ["c2", "c1", "c3_pre", "c3_post", "c4_dst7_pre", "c4_dct8_pre", "c4_dst7_post",
           "c4_dct8_post", "c5"]
C3_SIZES = np.array([16, 16, 32, 32])  # axis table: (16, dst7), (16, dct8), (32, dst7), (32, dct8)


# ------------------------------------------------------------------ sharding (host logic)
def c3_table():
    """Global config-3 block table: h_index, v_index into C3_SIZES and the
    coefficient count of every block (the weights of the equal-work split)."""
    from paper_2505_23618_b200 import workloads
    g_h, g_w, kinds = workloads._c3_table()
    h_kind, v_kind = (kinds % 2).numpy(), (kinds // 2).numpy()
    h_index = (np.where(g_w.numpy() == 16, 0, 2) + h_kind).astype(np.int32)
    v_index = (np.where(g_h.numpy() == 16, 0, 2) + v_kind).astype(np.int32)
    coefs = (C3_SIZES[h_index] * C3_SIZES[v_index]).astype(np.int64)
    return h_index, v_index, coefs


def shard_plan(cfg: str, rank: int, world: int, scaling: str = "strong") -> dict:
    """This rank's share of config `cfg`: {unit, total, start, stop, coefficients}.
    Strong scaling splits the config's total (C1/C2/C4: shard.block_range; C3:
    shard.weighted_ranges on coefficient counts; C5: shard.frame_range); weak
    scaling gives every rank the whole config."""
    from paper_2505_23618_b200 import shard, workloads
    if cfg in UNIFORM:
        total, n = UNIFORM[cfg][1], UNIFORM[cfg][2]
        s0, s1 = shard.block_range(rank, world, total) if scaling == "strong" else (0, total)
        return {"unit": "blocks", "total": total, "start": s0, "stop": s1,
                "coefficients": (s1 - s0) * n * n}
    if cfg.startswith("c3"):
        _, _, coefs = c3_table()
        s0, s1 = shard.weighted_ranges(coefs, world)[rank] if scaling == "strong" else (0, len(coefs))
        return {"unit": "blocks", "total": len(coefs), "start": s0, "stop": s1,
                "coefficients": int(coefs[s0:s1].sum())}
    if cfg == "c5":
        total = workloads.C5_FRAMES
        s0, s1 = shard.frame_range(rank, world, total) if scaling == "strong" else (0, total)
        per = -(-workloads.C5_HEIGHT // 32) * (workloads.C5_WIDTH // 32) * 1024
        return {"unit": "frames", "total": total, "start": s0, "stop": s1,
                "coefficients": (s1 - s0) * per}
    raise ValueError(f"unknown config {cfg!r}")


def n_sets(set_bytes: float, input_bytes: float) -> int:
    """Buffer sets the steps rotate over: two when the inputs exceed L2 -- consecutive
    steps are then independent batches, as a streaming caller double-buffers, and the
    library overlaps one step's tail with the next step's start (abi.cu pdl_early) --
    else enough sets that a full cycle moves >= 4x L2 (no step finds its inputs in
    L2).  The single-set schedule is measured beside it (`single_buffer_set`)."""
    if SETS_OVERRIDE > 0:
        return SETS_OVERRIDE
    if input_bytes > L2_BYTES:
        return 2
    return 1 + int(math.ceil(ROTATE_BYTES / max(set_bytes, 1.0)))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every
    ~0.5 ms while a timed region is open (mark_start .. mark_end); falls back to
    `nvidia-smi -lms 50` without NVML.  summary() covers the last region,
    summary(all=True) every region of the run."""

    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
            "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, torch_device: int):
        self.samples = []   # (region id, sm_mhz, reasons bitmask)
        self.region = -1
        self.active = False
        self._stop = False
        self.max_mhz = None
        self._h = None
        self.source = "nvml"
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = self._handle(torch_device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nv = None
            self.source = "nvidia-smi"
        self._dev = torch_device
        self._t = threading.Thread(target=self._run, daemon=True)

    def _handle(self, torch_device):
        import torch
        nv = self._nv
        try:
            uuid = str(torch.cuda.get_device_properties(torch_device).uuid)
            return nv.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [v for v in vis.split(",") if v.strip()]
            idx = int(ids[torch_device]) if torch_device < len(ids) and ids[torch_device].isdigit() \
                else torch_device
            return nv.nvmlDeviceGetHandleByIndex(idx)

    def _run(self):
        if self._nv is not None:
            nv = self._nv
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self._stop:
                if self.active:
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                        rs = get_r(self._h)
                        self.samples.append((self.region, float(sm), int(rs)))
                    except Exception:
                        pass
                    time.sleep(0.0005)
                else:
                    time.sleep(0.0002)
            return
        try:  # fallback: one long-running nvidia-smi
            proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self._dev), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._proc = proc
            bits = [0x8, 0x40, 0x20, 0x4]
            for line in proc.stdout:
                if self._stop:
                    break
                f = [x.strip() for x in line.split(",")]
                if self.active and len(f) >= 6 and f[0].replace(".", "", 1).isdigit():
                    self.max_mhz = float(f[1]) if f[1].replace(".", "", 1).isdigit() else self.max_mhz
                    rs = sum(b for b, v in zip(bits, f[2:6]) if v.lower() == "active")
                    self.samples.append((self.region, float(f[0]), rs))
        except Exception:
            pass

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop = True
        p = getattr(self, "_proc", None)
        if p is not None:
            p.terminate()
        self._t.join(timeout=5)

    def _sample_now(self):
        """One synchronous NVML sample (region boundaries: a region of a few ms can
        end before the polling thread is scheduled)."""
        if self._nv is None:
            return
        nv = self._nv
        try:
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            self.samples.append((self.region, float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)),
                                 int(get_r(self._h))))
        except Exception:
            pass

    def mark_start(self):
        """Called with the previous work drained, right before the first event of
        the region is recorded: samples the clocks as the region opens."""
        self.region += 1
        self._sample_now()
        self.active = True

    def sample_in_region(self):
        """A sample taken while the region's kernels are still queued / running."""
        self._sample_now()

    def mark_end(self):
        self._sample_now()
        self.active = False

    def summary(self, all_regions: bool = False) -> dict:
        win = [s for s in self.samples if all_regions or s[0] == self.region]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0, "source": self.source}
        sm = [s[1] for s in win]
        mask = 0
        for s in win:
            mask |= s[2]
        reasons = sorted(k for k, b in self.BITS.items() if mask & b)
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(win),
                "source": self.source}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(workload: str, launch: str):
    """ncu dram bytes (read + write) of one `launch` of `workload`, from
    profiles/ncu_traffic.json (keys "<workload>/<launch>")."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        return json.loads(p.read_text()).get(f"{workload}/{launch}")
    return None


def _merge_check(acc, r):
    if acc is None:
        return dict(r)
    out = dict(acc)
    out["blocks"] += r["blocks"]
    out["over_tol"] += r["over_tol"]
    if r["max_err"] > acc["max_err"]:
        out["max_err"] = r["max_err"]
    return out


# ------------------------------------------------------------------ GPU workloads
class Workload:
    """One config on one rank: R rotating buffer sets, the launches of one step,
    the full-shard oracle gate and (uniform configs) the host-buffer e2e step."""

    name = ""
    workload = ""
    dtype = "f32"
    launches: list = []          # [(name, fn(set index))] per step, in order
    two_kernel = None            # the same step as separate kernels (fused configs)
    coef_per_step = 0            # coefficients this rank produces per step
    bytes_first_launch = 0       # algorithmic bytes of launches[0]
    kernels_per_step = None      # device kernels launched per step (default: one per launch)
    kernel_name = "tile_kernel"
    nsets = 1
    e2e = None
    e2e_bytes = (0, 0)
    e2e_api = ""
    extra: dict = {}

    def step(self, i: int, launches=None):
        for _, fn in (launches or self.launches):
            fn(i % self.nsets)

    def gate(self, threads: int) -> dict:
        raise NotImplementedError

    def check_e2e(self):
        pass


class Uniform(Workload):
    def __init__(self, name: str, rank: int = 0, world: int = 1, scaling: str = "strong",
                 fused_roundtrip: bool = True, rotate: bool = True):
        import torch
        from paper_2505_23618_b200 import _lib, pipeline, workloads
        label, total, n, dt, make, inputs, inverse = UNIFORM[name]
        plan = shard_plan(name, rank, world, scaling)
        b0, b1 = plan["start"], plan["stop"]
        self.name, self.dtype, self.plan = name, dt, plan
        self.nblk = nblk = b1 - b0
        self.workload = f"{label}_{nblk}x{n}x{n}"
        self.t = make()
        self.inverse = inverse
        x = getattr(workloads, inputs)("cuda", nblk, offset=b0)
        es = x.element_size()
        coef = nblk * n * n
        nb = coef * es
        self.coef_per_step = coef * (2 if inverse else 1)
        self.bytes_first_launch = 2 * nb
        set_bytes = nb * (3 if inverse else 2)
        self.set_input_bytes = nb
        self.nsets = n_sets(set_bytes, nb) if rotate else 1
        self.sets = [{"x": x if s == 0 else x.clone(), "y": torch.empty_like(x),
                      "xr": torch.empty_like(x) if inverse else None} for s in range(self.nsets)]
        self.x, self.y, self.xr = self.sets[0]["x"], self.sets[0]["y"], self.sets[0]["xr"]
        lib = _lib.load()
        ax, self._keep = self.t.axis()
        self.ax = ax
        dtc = _lib.F32 if dt == "f32" else _lib.F64
        st = torch.cuda.current_stream().cuda_stream
        ref = ctypes.byref(ax)
        S = self.sets

        def fwd(s):
            _lib.check(lib.dctadj_forward_2d(ref, ref, S[s]["x"].data_ptr(), S[s]["y"].data_ptr(),
                                             nblk, dtc, st))

        def inv(s):
            _lib.check(lib.dctadj_inverse_2d(ref, ref, S[s]["y"].data_ptr(), S[s]["xr"].data_ptr(),
                                             nblk, dtc, st))

        def rt(s):  # forward + inverse in one kernel: x read once, y and x' written once
            _lib.check(lib.dctadj_roundtrip_2d(ref, ref, S[s]["x"].data_ptr(), S[s]["y"].data_ptr(),
                                               S[s]["xr"].data_ptr(), nblk, dtc, st))

        self.two_kernel = [("forward_2d", fwd)] + ([("inverse_2d", inv)] if inverse else [])
        self.launches = self.two_kernel
        if fused_roundtrip and inverse and lib.dctadj_roundtrip_fused(ref, ref, dtc):
            self.launches = [("roundtrip_2d", rt)]
            self.bytes_first_launch = 3 * nb
            self.kernel_name = "roundtrip_kernel"
        else:
            self.two_kernel = None
        # e2e: the same step through the host-buffer entries (pinned arrays)
        self.xh = x.cpu().pin_memory().numpy()
        self.yh = torch.empty(tuple(x.shape), dtype=x.dtype).pin_memory().numpy()
        self.xrh = torch.empty(tuple(x.shape), dtype=x.dtype).pin_memory().numpy()

        def e2e():
            if inverse:  # the round trip in one pipelined pass (coefficients D2H once)
                pipeline.roundtrip_adjusted_2d_host(self.t, self.t, self.xh, out=self.yh,
                                                    out_inv=self.xrh)
            else:
                pipeline.forward_adjusted_2d_host(self.t, self.t, self.xh, out=self.yh)

        self.e2e = e2e
        self.e2e_bytes = (nb, nb * (2 if inverse else 1))
        self.e2e_api = ("roundtrip_adjusted_2d_host (C-ABI dctadj_roundtrip_2d_host)" if inverse
                        else "forward_adjusted_2d_host (C-ABI dctadj_forward_2d_host)")
        self.extra = {"blocks_total": total, "blocks_this_rank": nblk, "block_range": [b0, b1],
                      "block": f"{n}x{n}"}

    def gate(self, threads: int) -> dict:
        """Every block of this rank's shard: y against the oracle on x, and (round
        trips) x' against the oracle's inverse on y; config 2 also the exact
        integer round trip rint(x') == x (SURVEY.md App. A D7 iii)."""
        import torch
        from oracle import oracle as O
        ax = _oaxis(self.t)
        tol = 1e-5 if self.dtype == "f32" else 1e-9
        per = max(1, GATE_CHUNK_BYTES // (self.x[0].numel() * self.x.element_size()))
        fwd = inv = None
        for c0 in range(0, self.nblk, per):
            c1 = min(self.nblk, c0 + per)
            xc = self.x[c0:c1].cpu().numpy()
            yc = self.y[c0:c1].cpu().numpy()
            fwd = _merge_check(fwd, O.check_2d(ax, ax, xc, yc, threads=threads, tol=tol))
            if self.inverse:
                xrc = self.xr[c0:c1].cpu().numpy()
                inv = _merge_check(inv, O.check_2d(ax, ax, yc, xrc, inverse=True, threads=threads,
                                                   tol=tol))
        out = {"tol": tol, "forward": fwd}
        if inv is not None:
            out["inverse"] = inv
        if self.name == "c2":
            out["integer_round_trip_exact"] = bool(torch.equal(torch.round(self.xr), self.x))
        return out

    def check_e2e(self):
        import torch
        torch.cuda.synchronize()
        if not np.array_equal(self.yh, self.y.cpu().numpy()):
            raise SystemExit("e2e coefficients differ from the device path")
        if self.inverse and not np.array_equal(self.xrh, self.xr.cpu().numpy()):
            raise SystemExit("e2e reconstruction differs from the device path")


class Mixed(Workload):
    """Config 3: 1,048,576 blocks, shapes {16,32}^2 and (h, v) kinds uniform;
    this rank's contiguous range at equal coefficient counts."""

    def __init__(self, side: str, rank: int = 0, world: int = 1, scaling: str = "strong",
                 fused_roundtrip: bool = True, rotate: bool = True):
        import torch
        from paper_2505_23618_b200 import _lib, pipeline, workloads
        self.name = f"c3_{side}"
        plan = shard_plan(self.name, rank, world, scaling)
        self.plan = plan
        b0, b1 = plan["start"], plan["stop"]
        gh, gv, coefs = c3_table()
        h_index, v_index = gh[b0:b1], gv[b0:b1]
        nblk = b1 - b0
        self.workload = f"c3_mixed_{side}_fwd+inv_{nblk}blocks"
        self.batch = pipeline.MixedBatch.packed(h_index, v_index, C3_SIZES)
        if side == "pre":
            self.table = [_pre(16, "dst7"), _pre(16, "dct8"), _pre(32, "dst7"), _pre(32, "dct8")]
        else:
            self.table = [_post(16, "dst7"), _post(16, "dct8"), _post(32, "dst7"), _post(32, "dct8")]
        total = self.batch.total_elements
        x = torch.empty(total, device="cuda", dtype=torch.float32)
        workloads.c3_fill(x, self.batch.offsets, b0)
        nb = total * 4
        self.set_input_bytes = nb
        self.nsets = n_sets(3 * nb, nb) if rotate else 1
        self.sets = [{"x": x if s == 0 else x.clone(), "y": torch.empty_like(x),
                      "xr": torch.empty_like(x)} for s in range(self.nsets)]
        self.x, self.y, self.xr = self.sets[0]["x"], self.sets[0]["y"], self.sets[0]["xr"]
        self.coef_per_step = 2 * total
        self.bytes_first_launch = 2 * nb
        self.axes = (_lib.Axis * 4)()
        self._keep = []
        for k, tr in enumerate(self.table):
            ax, m = tr.axis()
            self.axes[k] = ax
            self._keep.append(m)
        lib = _lib.load()
        st = torch.cuda.current_stream().cuda_stream
        planp = self.batch._plan
        S = self.sets

        def fwd(s):
            _lib.check(lib.dctadj_mixed_forward(planp, self.axes, S[s]["x"].data_ptr(),
                                                S[s]["y"].data_ptr(), 0, st))

        def inv(s):
            _lib.check(lib.dctadj_mixed_inverse(planp, self.axes, S[s]["y"].data_ptr(),
                                                S[s]["xr"].data_ptr(), 0, st))

        def rt(s):  # one fused gather kernel per class: x read once, y and x' written once
            _lib.check(lib.dctadj_mixed_roundtrip(planp, self.axes, S[s]["x"].data_ptr(),
                                                  S[s]["y"].data_ptr(), S[s]["xr"].data_ptr(), 0, st))

        self.two_kernel = [("mixed_forward", fwd), ("mixed_inverse", inv)]
        self.launches = self.two_kernel
        nclass = len(np.unique(np.asarray(h_index) * 4 + np.asarray(v_index)))
        self.kernels_per_step = 2 * nclass
        if fused_roundtrip and lib.dctadj_mixed_roundtrip_fused(planp, self.axes, 0):
            self.launches = [("mixed_roundtrip", rt)]
            self.kernels_per_step = nclass
            self.bytes_first_launch = 3 * nb
            self.kernel_name = "roundtrip_kernel (gather, one per class)"
        else:
            self.two_kernel = None
        self.h_index, self.v_index = h_index, v_index
        self.extra = {"blocks_total": len(coefs), "blocks_this_rank": nblk, "block_range": [b0, b1],
                      "coefficients_this_rank": total, "classes": int(nclass)}

    def gate(self, threads: int) -> dict:
        from oracle import oracle as O
        table = [_oaxis(t) for t in self.table]
        offs = self.batch.offsets
        n = self.batch.nblk
        ends = np.append(offs[1:], self.batch.total_elements)
        fwd = inv = None
        i0 = 0
        while i0 < n:
            i1 = int(np.searchsorted(ends, offs[i0] + GATE_CHUNK_BYTES // 4, side="right"))
            i1 = max(i0 + 1, min(n, i1))
            e0, e1 = int(offs[i0]), int(ends[i1 - 1])
            xc = self.x[e0:e1].cpu().numpy()
            yc = self.y[e0:e1].cpu().numpy()
            xrc = self.xr[e0:e1].cpu().numpy()
            o = offs[i0:i1] - e0
            hi, vi = self.h_index[i0:i1], self.v_index[i0:i1]
            fwd = _merge_check(fwd, O.check_mixed(table, hi, vi, o, xc, yc, threads=threads,
                                                  tol=1e-5))
            inv = _merge_check(inv, O.check_mixed(table, hi, vi, o, yc, xrc, inverse=True,
                                                  threads=threads, tol=1e-5))
            i0 = i1
        return {"tol": 1e-5, "forward": fwd, "inverse": inv}


class Frames(Workload):
    """Config 5: 3840x2160 fp32 frames (this rank's frame range), 32x32 tiles
    (bottom padded to 2176 rows by TMA zero fill); adjusted DST-7 (sub8 post)
    forward + inverse plus the exact dense DST-7 forward on the same tiles.  The
    coefficient-domain approximation error sum|Y_adj - Y_exact|^2 /
    sum|Y_exact|^2 is reported over all tiles and over the 67 unpadded tile rows."""

    def __init__(self, rank: int = 0, world: int = 1, scaling: str = "strong", rotate: bool = True):
        import torch
        from paper_2505_23618_b200 import _lib, pipeline, workloads
        from paper_2505_23618_b200.design import (AdjustmentMatrix, Side, SparsityPattern,
                                                  pattern_schedule_template)
        from paper_2505_23618_b200.transforms import TransformKind, build_transform
        self.name = "c5"
        plan = shard_plan("c5", rank, world, scaling)
        self.plan = plan
        f0, f1 = plan["start"], plan["stop"]
        self.nframes = F = f1 - f0
        self.H, self.W = H, W = workloads.C5_HEIGHT, workloads.C5_WIDTH
        self.workload = f"c5_frames_{F}x3840x2160_dst7_post_sub8_fwd+inv+dense_exact"
        frames = workloads.c5_frames(F, H, W, offset=f0)
        self.t = _post(32, "dst7")
        d7 = build_transform(TransformKind.DST7, 32).entries
        c = d7 @ build_transform(TransformKind.DCT2, 32).entries.T
        dense = AdjustmentMatrix(SparsityPattern.dense(32), Side.POST, TransformKind.DCT2,
                                 TransformKind.DST7, pattern_schedule_template(SparsityPattern.dense(32)), c)
        self.td = pipeline.make_adjusted_transform(dense)
        nblk = pipeline.frame_block_count(F, H, W, 32, 32)
        self.nblk = nblk
        nb = F * H * W * 4
        coef = nblk * 1024
        self.set_input_bytes = nb
        self.nsets = n_sets(nb + 2 * coef * 4 + nb, nb) if rotate else 1
        self.sets = [{"frames": frames if s == 0 else frames.clone(),
                      "y": torch.empty(nblk, 32, 32, device="cuda"),
                      "ye": torch.empty(nblk, 32, 32, device="cuda"),
                      "back": torch.empty_like(frames),
                      "err": torch.zeros((F, 4), dtype=torch.float64, device="cuda")}
                     for s in range(self.nsets)]
        s0 = self.sets[0]
        self.frames, self.y, self.ye, self.back, self.err = (s0["frames"], s0["y"], s0["ye"],
                                                             s0["back"], s0["err"])
        lib = _lib.load()
        st = torch.cuda.current_stream().cuda_stream
        (ax, k1), (axd, k2) = self.t.axis(), self.td.axis()
        self._keep = (ax, k1, axd, k2)
        r, rd = ctypes.byref(ax), ctypes.byref(axd)
        S = self.sets

        def fwd(s):
            _lib.check(lib.dctadj_forward_frames(r, r, S[s]["frames"].data_ptr(), S[s]["y"].data_ptr(),
                                                 F, H, W, 0, st))

        def inv(s):
            _lib.check(lib.dctadj_inverse_frames(r, r, S[s]["y"].data_ptr(), S[s]["back"].data_ptr(),
                                                 F, H, W, 0, st))

        def dense_fwd(s):
            _lib.check(lib.dctadj_forward_frames(rd, rd, S[s]["frames"].data_ptr(),
                                                 S[s]["ye"].data_ptr(), F, H, W, 0, st))

        def fwd_exact(s):  # adjusted + exact forward and the error sums, one read of the frames
            _lib.check(lib.dctadj_forward_frames_exact(r, r, rd, rd, S[s]["frames"].data_ptr(),
                                                       S[s]["y"].data_ptr(), S[s]["ye"].data_ptr(),
                                                       S[s]["err"].data_ptr(), F, H, W, 0, st))

        self.launches = [("forward_frames_exact", fwd_exact), ("inverse_frames", inv)]
        self.kernel_name = "dense_tc_kernel<FRAME4, FUSED sub8-post>"
        # the same three transforms as separate kernels (error sums not included)
        self.two_kernel = [("forward_frames", fwd), ("dense_dst7_frames", dense_fwd),
                           ("inverse_frames", inv)]
        self.coef_per_step = 3 * coef
        self.bytes_first_launch = nb + 2 * coef * 4
        self.extra = {"frames_total": plan["total"], "frames_this_rank": F, "frame_range": [f0, f1],
                      "blocks_this_rank": nblk, "padded_rows": 2176,
                      "coefficients_padded": coef, "coefficients_unpadded": F * H * W,
                      "step": "fused [adjusted DST-7 forward + exact dense DST-7 forward + per-frame "
                              "error sums] (one read of the frames) + adjusted inverse; value counts "
                              "all three transforms"}

    def gate(self, threads: int) -> dict:
        """Every tile of this rank's frames: adjusted forward, exact dense forward
        and the adjusted inverse (rows inside the frame) against the oracle."""
        from oracle import oracle as O
        ax, axd = _oaxis(self.t), _oaxis(self.td)
        per_frame = self.nblk // max(1, self.nframes)
        fwd = ex = inv = None
        step = max(1, GATE_CHUNK_BYTES // (self.H * self.W * 4))
        for f0 in range(0, self.nframes, step):
            f1 = min(self.nframes, f0 + step)
            fr = self.frames[f0:f1].cpu().numpy()
            yc = self.y[f0 * per_frame:f1 * per_frame].cpu().numpy()
            yec = self.ye[f0 * per_frame:f1 * per_frame].cpu().numpy()
            bc = self.back[f0:f1].cpu().numpy()
            fwd = _merge_check(fwd, O.check_frames(ax, ax, fr, yc, threads=threads, tol=1e-5))
            ex = _merge_check(ex, O.check_frames(axd, axd, fr, yec, threads=threads, tol=1e-5))
            inv = _merge_check(inv, O.check_frames(ax, ax, bc, yc, inverse=True, threads=threads,
                                                   tol=1e-5))
        return {"tol": 1e-5, "forward": fwd, "exact_dense_forward": ex, "inverse": inv}

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


def make_workload(cfg: str, rank: int, world: int, scaling: str, fused: bool = True) -> Workload:
    if cfg in UNIFORM:
        return Uniform(cfg, rank, world, scaling, fused_roundtrip=fused)
    if cfg.startswith("c3"):
        return Mixed(cfg.split("_")[1], rank, world, scaling, fused_roundtrip=fused)
    return Frames(rank, world, scaling)


# ------------------------------------------------------------------ CPU legs
_REF_X = None      # the C2 array, shared with the fork-pool workers
_REF_PIPE = None   # (forward_2d, inverse_2d, kind, source)


def reference_pipeline():
    """The reference's CPU path for config 2, best available:
    1. the reference package itself (oracle/_ref/pkg, compiled backend) through
       its public API (make_adjusted_transform / forward_adjusted /
       inverse_adjusted, rows then columns as BASELINE.md 3.3) -- kind "reference";
    2. the reference's compiled core (oracle/_ref/_fastcore) under the restated
       policy layer (oracle.RefPipeline) -- kind "reference";
    3. the C restatement (oracle/liboracle.so) -- kind "port"."""
    global _REF_PIPE
    if _REF_PIPE is not None:
        return _REF_PIPE
    from oracle import oracle as O
    pkg = ROOT / "oracle" / "_ref" / "pkg" / "src"
    adj_file = ROOT / "paper_2505_23618_b200" / "adjustments" / "sub8_post_dct2_dst7_n32.adj"
    if (pkg / "dctadjust").is_dir():
        try:
            os.environ["DCTADJUST_BACKEND"] = "compiled"
            sys.path.insert(0, str(pkg))
            from dctadjust import design as rdesign, kernels as rkernels, matio as rmatio
            from dctadjust import pipeline as rpipe
            if rkernels.BACKEND != "compiled":
                raise ImportError("reference compiled core not built")
            t = rpipe.make_adjusted_transform(
                rdesign.dct8_adjustment_from_dst7(rmatio.read_adjustment(str(adj_file))))

            def fwd(x):
                b, h, w = x.shape
                rows = rpipe.forward_adjusted(t, x.reshape(b * h, w)).reshape(b, h, w)
                cols = np.ascontiguousarray(rows.transpose(0, 2, 1)).reshape(b * w, h)
                return np.ascontiguousarray(rpipe.forward_adjusted(t, cols).reshape(b, w, h)
                                            .transpose(0, 2, 1))

            def inv(y):
                b, h, w = y.shape
                cols = np.ascontiguousarray(y.transpose(0, 2, 1)).reshape(b * w, h)
                t2 = np.ascontiguousarray(rpipe.inverse_adjusted(t, cols).reshape(b, w, h)
                                          .transpose(0, 2, 1))
                return rpipe.inverse_adjusted(t, t2.reshape(b * h, w)).reshape(b, h, w)

            _REF_PIPE = (fwd, inv, "reference", "reference package dctadjust (oracle/_ref/pkg, "
                         "compiled backend): forward_adjusted / inverse_adjusted, rows then columns")
            return _REF_PIPE
        except Exception:
            pass
    from paper_2505_23618_b200 import matio
    from paper_2505_23618_b200.design import dct8_adjustment_from_dst7
    a8 = dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32"))
    oax = O.OAxis(32, O.BASE_DCT2, O.ADJ_SUBBLOCK, O.SIDE_POST, 0, 8, np.array(a8.realized))
    if O.ref_fastcore() is not None:
        ref = O.RefPipeline()
        _REF_PIPE = (lambda x: ref.forward_2d(oax, oax, x), lambda y: ref.inverse_2d(oax, oax, y),
                     "reference", "reference compiled core (oracle/_ref/_fastcore) + restated policy layer")
    else:
        _REF_PIPE = (lambda x: O.adjusted_2d(oax, oax, x), lambda y: O.adjusted_2d(oax, oax, y, inverse=True),
                     "port", "C restatement (oracle/liboracle.so)")
    return _REF_PIPE


def _ref_worker(args):
    b0, b1, reps = args
    fwd, inv, _, _ = reference_pipeline()
    x = _REF_X[b0:b1].astype(np.float64)
    t0 = time.perf_counter()
    for _ in range(reps):
        inv(fwd(x))
    return time.perf_counter() - t0


class RefPool:
    """The reference CPU path over the full config-2 array, one contiguous block
    range per host core (fork pool, single-threaded BLAS)."""

    def __init__(self):
        global _REF_X
        from multiprocessing import get_context
        from oracle import oracle as O
        from paper_2505_23618_b200 import shard, workloads
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        os.environ["OMP_NUM_THREADS"] = "1"
        _REF_X = workloads.c2_inputs_host()
        self.nblk = _REF_X.shape[0]
        self.coef_per_pass = 2 * _REF_X.size
        _, _, self.kind, self.source = reference_pipeline()
        self.cores = O.threads_available()
        self.ranges = [shard.block_range(r, self.cores, self.nblk) for r in range(self.cores)]
        self.pool = get_context("fork").Pool(self.cores)

    def run(self, reps: int = 1) -> float:
        """Wall seconds for `reps` passes (forward + inverse) over the whole array."""
        t0 = time.perf_counter()
        self.pool.map(_ref_worker, [(b0, b1, reps) for b0, b1 in self.ranges])
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, reps: int) -> str:
        return (f"{reps} pass(es) of forward + inverse over the full config-2 array "
                f"(65,536 x 32x32, the same seeded input as the GPU arm), "
                f"{self.cores} processes x one contiguous block range each; {self.source}")


def cpu_baseline(wall_target: float = 2.0) -> dict:
    """cpu_baseline leg (rank 0, N=1): ~wall_target s of all-core work (~30 core-s)."""
    rp = RefPool()
    try:
        t1 = rp.run(1)  # warm
        reps = max(1, min(20, int(round(wall_target / max(t1, 1e-3)))))
        dt = rp.run(reps)
        value = reps * rp.coef_per_pass / dt
        return {"value": value, "unit": UNIT, "cores": rp.cores, "kind": rp.kind,
                "sample": rp.describe(reps)}
    finally:
        rp.close()


def run_reference(args, rank: int, world: int):
    """`--impl reference`: the reference's CPU path alone on config 2 (rank 0; the
    other ranks exit): every step is one pass of forward + inverse over the full
    65,536-block array on all host cores."""
    if rank != 0:
        return
    rp = RefPool()
    try:
        for _ in range(args.warmup):
            rp.run(1)
        per = [rp.run(1) for _ in range(args.steps)]
    finally:
        rp.close()
    total = float(sum(per))
    value = args.steps * rp.coef_per_pass / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (the GPU arm's seeded config-2 array, workloads.c2_inputs_host)",
            "impl": "reference",
            "config": {"workload": UNIFORM["c2"][0] + "_65536x32x32", "median_step_ms":
                       float(np.median(per)) * 1e3},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": rp.cores, "kind": rp.kind,
                             "sample": rp.describe(1) + " per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def _time_launch(stream, fn, nsets: int, reps: int) -> float:
    import torch
    fn(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(reps):
        fn(i % nsets)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def measure(w: Workload, args, rank: int, world: int, clk: ClockSampler, threads: int) -> dict:
    """Gate, warm up, time K steps (max over ranks), per-launch durations, e2e."""
    import torch
    import torch.distributed as dist
    from paper_2505_23618_b200 import shard
    stream = torch.cuda.current_stream()
    w.step(0)
    torch.cuda.synchronize()
    # oracle gate over the whole shard before timing (reference benchmark.py:181-190)
    gate = w.gate(threads)
    worst = max(v["max_err"] for v in gate.values() if isinstance(v, dict))
    bad = int(not (worst <= gate["tol"])) + int(gate.get("integer_round_trip_exact") is False)
    if world > 1:
        t = torch.tensor([float(bad)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        bad = int(t.item())
    if bad:
        raise SystemExit(f"oracle gate failed on {w.name} (rank {rank}): {json.dumps(gate)}")

    # warm-up: at least W steps, and at least ~50 ms of GPU work so short steps (config
    # 1: ~15 us) do not time a GPU still ramping out of the idle gate phase
    t0 = time.perf_counter()
    i = 0
    while i < args.warmup or time.perf_counter() - t0 < 0.05:
        w.step(i)
        i += 1
        if i % 32 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    for key in ("y", "xr", "ye", "back"):
        t = getattr(w, key, None)
        if t is not None and not bool(torch.isfinite(t).all()):
            raise SystemExit(f"non-finite values in {key} after the warm-up steps ({w.name})")

    # timed region: K steps back to back, CUDA events only at its two ends (an
    # event between launches would serialise the kernels' programmatic launch)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.mark_start()
    e0.record(stream)
    for i in range(args.steps):
        w.step(i)
    e1.record(stream)
    clk.sample_in_region()  # the launches are queued: the GPU is running them now
    torch.cuda.synchronize()
    clk.mark_end()
    if world > 1:
        dist.barrier()
    total_ms = e0.elapsed_time(e1)
    clocks = clk.summary()

    # per-kernel durations (roofline): each launch type back to back on the same
    # stream over the rotating sets, CUDA events around the run
    reps = max(10, min(args.steps, 200))
    per_launch_ms = [_time_launch(stream, fn, w.nsets, reps) for _, fn in w.launches]
    unfused = None
    if w.two_kernel:
        ums = [_time_launch(stream, fn, w.nsets, reps) for _, fn in w.two_kernel]
        unfused = {"value_this_rank": w.coef_per_step / (sum(ums) / 1e3),
                   "per_launch_ms": dict(zip([n for n, _ in w.two_kernel], ums)),
                   "note": "the same transforms as separate kernels, each reading its input "
                           "from HBM"}
    # dispersion: per-step CUDA events over up to 50 further steps (median, IQR)
    nsamp = min(args.steps, 50)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(nsamp + 1)]
    ev[0].record(stream)
    for i in range(nsamp):
        w.step(i)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    step_ms = np.array([ev[i].elapsed_time(ev[i + 1]) for i in range(nsamp)])
    q1, med, q3 = np.percentile(step_ms, [25, 50, 75])
    resident = None
    if w.nsets > 1:  # the same steps on ONE buffer set, for reference: each step writes the
        # previous step's outputs again, so it waits for it (no cross-launch overlap);
        # inputs L2-resident when a set fits L2
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            w.step(0)
        b.record(stream)
        torch.cuda.synchronize()
        resident = a.elapsed_time(b) / args.steps

    e2e_ms = 0.0
    if w.e2e is not None:
        w.e2e()  # warm
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n_e2e = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            w.e2e()
        e2e_ms = (time.perf_counter() - t0) / n_e2e * 1e3
        w.check_e2e()

    approx = w.approximation_error() if isinstance(w, Frames) else [0.0, 0.0, 0.0, 0.0]
    st = shard.reduce_stats(shard.Stats(
        elapsed_ms=total_ms, e2e_ms=e2e_ms, coefficients=w.coef_per_step,
        err_energy=approx[0], ref_energy=approx[1], err_energy_full=approx[2],
        ref_energy_full=approx[3], max_rel_err=worst), device="cuda")
    ms_per_step = st.elapsed_ms / args.steps
    peak, peak_src = _peaks()
    achieved = w.bytes_first_launch / (per_launch_ms[0] / 1e3) / 1e9
    res = {
        "workload": w.workload, "value": st.coefficients / (ms_per_step / 1e3),
        "ms_per_step": ms_per_step, "coefficients_per_step": st.coefficients,
        "kernels_per_step": w.kernels_per_step or len(w.launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic(w.workload, w.launches[0][0]),
                     "peak_source": peak_src, "kernel": f"{w.kernel_name} ({w.launches[0][0]})",
                     "algorithmic_bytes_per_launch": w.bytes_first_launch,
                     "avg_launch_ms": per_launch_ms[0],
                     "per_launch_ms": dict(zip([n for n, _ in w.launches], per_launch_ms)),
                     "measured_on": f"rank {rank}'s shard"},
        "gate": gate, "gate_max_rel_err_all_ranks": st.max_rel_err, "clocks": clocks,
        "dispersion": {"median_ms_per_step": float(med), "iqr_ms": float(q3 - q1),
                       "samples": nsamp, "note": "this rank, per-step events after the timed region"},
        "l2": (f"{w.nsets} rotating buffer sets (cycle > 4x the 126 MB L2)"
               if w.set_input_bytes <= L2_BYTES else
               f"inputs > 126 MB L2 per rank; {w.nsets} buffer sets alternate (independent "
               "consecutive batches: double buffering)"),
        "shard": w.plan, "schedule": ", ".join(n for n, _ in w.launches),
    }
    res.update({"extra": w.extra})
    if unfused is not None:
        res["unfused_separate_kernels"] = unfused
    if resident is not None:
        res["single_buffer_set"] = {
            "ms_per_step": resident, "value_this_rank": w.coef_per_step / (resident / 1e3),
            "note": ("one buffer set, steps serialised by their shared outputs; inputs "
                     + ("L2-resident" if w.set_input_bytes <= L2_BYTES else "> 126 MB L2, from HBM"))}
    if w.e2e is not None:
        res["e2e"] = {"value": st.coefficients / (st.e2e_ms / 1e3), "unit": UNIT,
                      "h2d_bytes_per_step": w.e2e_bytes[0] * world,
                      "d2h_bytes_per_step": w.e2e_bytes[1] * world, "api": w.e2e_api,
                      "ms_per_step": st.e2e_ms}
    if isinstance(w, Frames):
        res["approx_error_vs_exact_dst7_all_tiles"] = st.err_energy / st.ref_energy
        res["approx_error_vs_exact_dst7_unpadded_tile_rows"] = st.err_energy_full / st.ref_energy_full
    return res


def _brief(r: dict) -> dict:
    """per_config entry: the numbers the verdict asks for, per config."""
    g = r["gate"]
    out = {"workload": r["workload"], "value": r["value"], "ms_per_step": r["ms_per_step"],
           "frac": r["roofline"]["frac"], "kernel": r["roofline"]["kernel"],
           "traffic": r["roofline"]["traffic"],
           "algorithmic_bytes_per_launch": r["roofline"]["algorithmic_bytes_per_launch"],
           "avg_launch_ms": r["roofline"]["avg_launch_ms"],
           "per_launch_ms": r["roofline"]["per_launch_ms"],
           "gate": {k: (v if not isinstance(v, dict) else
                        {"max_err": v["max_err"], "blocks": v["blocks"], "over_tol": v["over_tol"]})
                    for k, v in g.items()},
           "clocks": r["clocks"], "l2": r["l2"], "schedule": r["schedule"]}
    for k in ("unfused_separate_kernels", "single_buffer_set", "e2e",
              "approx_error_vs_exact_dst7_all_tiles", "approx_error_vs_exact_dst7_unpadded_tile_rows"):
        if k in r:
            out[k] = r[k]
    return out


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist
    from oracle import oracle as O

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    threads = max(1, O.threads_available() // world)
    order = [args.config] + ([c for c in CONFIGS if c != args.config] if args.per_config else [])
    results = {}
    with ClockSampler(local_rank) as clk:
        for cfg in order:
            if cfg != order[0] and world == 1 and not INPROC:
                # every other config in a fresh process: measured in-process after the
                # headline and the configs before it, the large ones lost 5-10 %
                # (C4 post 1.34-1.42 -> 1.52-1.57 ms per launch, C5 fused 1.36-1.39 ->
                # 1.46-1.50 ms) -- allocator / memory-placement state, not temperature
                results[cfg] = _measure_in_child(cfg, args)
                continue
            w = make_workload(cfg, rank, world, args.scaling, fused=not args.unfused)
            torch.cuda.synchronize()
            results[cfg] = measure(w, args, rank, world, clk, threads)
            head = results[cfg] if cfg == args.config else None
            if head is not None:
                gpu_launches = args.steps * (w.kernels_per_step or len(w.launches))
                dtype = w.dtype
            del w
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
        run_clocks = clk.summary(all_regions=True)

    h = results[args.config]
    config = {"workload": h["workload"], "parallelism": f"{args.scaling} scaling, "
              f"{h['shard']['unit']} split over {world} rank(s), no data-path collective",
              "shard_this_rank": h["shard"], "gate": h["gate"],
              "gate_max_rel_err_all_ranks": h["gate_max_rel_err_all_ranks"], "l2": h["l2"],
              "schedule": h["schedule"]}
    config.update(h["extra"])
    for k in ("unfused_separate_kernels", "single_buffer_set",
              "approx_error_vs_exact_dst7_all_tiles", "approx_error_vs_exact_dst7_unpadded_tile_rows"):
        if k in h:
            config[k] = h[k]
    if args.per_config:
        config["per_config"] = {cfg: _brief(results[cfg]) for cfg in order}
    clocks = dict(h["clocks"])
    clocks["run"] = run_clocks
    line = {
        "metric": METRIC, "value": h["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": h["ms_per_step"], "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (seeded residual fields per BASELINE.json configs, SURVEY.md App. A D12)",
        "config": config, "roofline": h["roofline"], "e2e": h.get("e2e"),
        "gpu_launches": gpu_launches, "clocks": clocks, "dispersion": h["dispersion"],
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ launch
def dry_run(args, rank: int, world: int):
    """Host logic only (no GPU): every rank's shard of every config, gathered
    over gloo, and the post-timing scalar reduction; rank 0 prints the plan."""
    import torch.distributed as dist
    from paper_2505_23618_b200 import shard
    if world > 1:
        dist.init_process_group("gloo")
    plans = {cfg: shard_plan(cfg, rank, world, args.scaling) for cfg in CONFIGS}
    gathered = [None] * world
    if world > 1:
        dist.all_gather_object(gathered, plans)
    else:
        gathered = [plans]
    st = shard.reduce_stats(shard.Stats(elapsed_ms=float(rank + 1),
                                        coefficients=plans["c2"]["coefficients"]))
    if rank == 0:
        out = {"dry_run": True, "world": world, "scaling": args.scaling,
               "ranges": {cfg: [g[cfg]["start"] for g in gathered] + [gathered[-1][cfg]["stop"]]
                          for cfg in CONFIGS},
               "per_rank": {cfg: [[g[cfg]["start"], g[cfg]["stop"]] for g in gathered] for cfg in CONFIGS},
               "totals": {cfg: plans[cfg]["total"] for cfg in CONFIGS},
               "coefficients": {cfg: sum(g[cfg]["coefficients"] for g in gathered) for cfg in CONFIGS},
               "reduced": {"elapsed_ms_max": st.elapsed_ms, "c2_coefficients_sum": st.coefficients}}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _measure_in_child(cfg: str, args) -> dict:
    """measure() of one config in a fresh process (world 1): `--measure-only`."""
    cmd = [sys.executable, str(Path(__file__).resolve()), "--measure-only", cfg,
           "--steps", str(args.steps), "--warmup", str(args.warmup), "--scaling", args.scaling]
    if args.unfused:
        cmd.append("--unfused")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith('{"measure"')]
    if out.returncode != 0 or not lines:
        raise SystemExit(f"per_config {cfg}: child failed (rc {out.returncode}): "
                         f"{out.stderr[-1500:]}")
    return json.loads(lines[-1])["measure"]


def run_measure_only(args):
    """The child of _measure_in_child: one config, its measure() dict as JSON."""
    import torch
    from oracle import oracle as O
    torch.cuda.set_device(0)
    with ClockSampler(0) as clk:
        w = make_workload(args.measure_only, 0, 1, args.scaling, fused=not args.unfused)
        torch.cuda.synchronize()
        res = measure(w, args, 0, 1, clk, max(1, O.threads_available()))
    res["kernels_per_step_launches"] = w.kernels_per_step or len(w.launches)
    print(json.dumps({"measure": res}), flush=True)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=CONFIGS)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-per-config", dest="per_config", action="store_false",
                    help="measure only --config (default: every BASELINE config, per_config)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--unfused", action="store_true",
                    help="fwd+inv configs: time forward and inverse as two kernels instead of "
                         "the fused round trip")
    ap.add_argument("--cpu-seconds", type=float, default=2.0,
                    help="cpu_baseline: wall seconds of all-core reference work")
    ap.add_argument("--dry-run", action="store_true",
                    help="host logic only: print every rank's shard plan (gloo, no GPU)")
    ap.add_argument("--measure-only", choices=CONFIGS, default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3 and not args.dry_run:
        ap.error("--warmup must be >= 3")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU, launched exactly as the driver does
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("OMP_NUM_THREADS", "1")
        sys.exit(subprocess.run(cmd, env=env).returncode)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and not args.dry_run:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}; using {world}", file=sys.stderr)
    if args.dry_run:
        dry_run(args, rank, world)
    elif args.measure_only:
        run_measure_only(args)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

"""Seeded synthetic inputs for the five BASELINE.json configurations.

No dataset is involved (the paper's VVC test sequences are neither available
nor needed): each config's residuals are generated with the shapes, sizes and
value distributions BASELINE.json states, following SURVEY.md App. A D12-D13.
Generation is plumbing, outside every timed region; the CPU oracle sees the
very same arrays (copied back from the device).

Every generator is SHARD-INVARIANT: the global array is defined in fixed
chunks of blocks (or per frame), each from its own seed, and a call for the
block range [offset, offset + nblk) returns exactly that slice of the global
array -- so a config split over 1, 2, 4 or 8 ranks processes the same data.

  C1  4,096 x 32x32 fp64, separable Gaussian AR(1) rho=0.9, sigma=32, seed 1
  C2  65,536 x 32x32 fp32, AR(1) rho=0.85, sigma=24, rint + clip [-512, 511], seed 2
      (host numpy, default_rng([2, chunk]) -- the reference arm reads the same array)
  C3  1,048,576 blocks, shapes {16,32}^2, Laplace(b=16) innovations mixed by AR(1) 0.9, seed 3
  C4  262,144 x 64x64 fp32, AR(1) rho=0.95, sigma=40, seed 4
  C5  64 frames 3840x2160 fp32, row/column AR(1) recursion rho_h=0.92, rho_v=0.88, sigma=30, seed 5
"""
from __future__ import annotations

import math

import numpy as np
import torch

CHUNK = 4096  # blocks per seeded chunk (C1, C2, C3, C4)

C1_BLOCKS, C2_BLOCKS, C3_BLOCKS, C4_BLOCKS = 4096, 65536, 1 << 20, 262144
C5_FRAMES, C5_HEIGHT, C5_WIDTH = 64, 2160, 3840


def ar1_chol(n: int, rho: float, device, dtype=torch.float64) -> torch.Tensor:
    i = torch.arange(n, device=device, dtype=torch.float64)
    k = rho ** (i[:, None] - i[None, :]).abs()
    return torch.linalg.cholesky(k).to(dtype)


def _chunks(offset: int, nblk: int, chunk: int):
    """(chunk index, first block of the chunk wanted, last + 1, destination start)"""
    g0, g1 = offset, offset + nblk
    for k in range(g0 // chunk, (g1 + chunk - 1) // chunk):
        c0, c1 = max(g0, k * chunk), min(g1, (k + 1) * chunk)
        yield k, c0 - k * chunk, c1 - k * chunk, c0 - g0


def ar1_blocks(nblk: int, h: int, w: int, rho: float, sigma: float, seed: int, device="cuda",
               dtype=torch.float32, chunk: int = CHUNK, offset: int = 0) -> torch.Tensor:
    """Blocks [offset, offset + nblk) of the global array sigma * L_v Z L_h^T,
    Z ~ N(0, 1) i.i.d.; chunk k of `chunk` blocks drawn from seed (seed, k)."""
    out = torch.empty(nblk, h, w, device=device, dtype=dtype)
    lv = ar1_chol(h, rho, device, torch.float32)
    lh = ar1_chol(w, rho, device, torch.float32)
    for k, a, b, d in _chunks(offset, nblk, chunk):
        g = torch.Generator(device=device).manual_seed(seed * 1_000_003 + k)
        z = torch.randn(chunk, h, w, device=device, generator=g)[a:b]
        out[d:d + (b - a)] = (sigma * (lv @ z @ lh.T)).to(dtype)
    return out


def c1_inputs(device="cuda", nblk: int = C1_BLOCKS, offset: int = 0) -> torch.Tensor:
    return ar1_blocks(nblk, 32, 32, 0.9, 32.0, 1, device, torch.float64, offset=offset)


def c2_inputs_host(nblk: int = C2_BLOCKS, offset: int = 0) -> np.ndarray:
    """Config 2 on the host (numpy, fp64 generation -> exact integers in fp32):
    chunk k from default_rng([2, k]).  Both bench arms
    (ours and the reference's CPU path) process this very array."""
    out = np.empty((nblk, 32, 32), dtype=np.float32)
    i = np.arange(32)
    lc = np.linalg.cholesky(0.85 ** np.abs(i[:, None] - i[None, :]))
    for k, a, b, d in _chunks(offset, nblk, CHUNK):
        z = np.random.default_rng([2, k]).standard_normal((CHUNK, 32, 32))[a:b]
        out[d:d + (b - a)] = np.clip(np.rint(24.0 * (lc @ z @ lc.T)), -512, 511)
    return out


def c2_inputs(device="cuda", nblk: int = C2_BLOCKS, offset: int = 0) -> torch.Tensor:
    return torch.from_numpy(c2_inputs_host(nblk, offset)).to(device)


def c4_inputs(device="cuda", nblk: int = C4_BLOCKS, offset: int = 0) -> torch.Tensor:
    return ar1_blocks(nblk, 64, 64, 0.95, 40.0, 4, device, torch.float32, offset=offset)


def c3_shapes(nblk: int = C3_BLOCKS, seed: int = 3) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Per-block (H, W) uniform over {16x16, 16x32, 32x16, 32x32} (H x W read, D9)
    and per-block (h, v) kinds uniform over {DST-7 = 0, DCT-8 = 1}^2 (CPU tensors)
    for the whole config (every rank draws the same global table)."""
    g = torch.Generator().manual_seed(seed * 7919 + 1)
    shape = torch.randint(0, 4, (nblk,), generator=g)
    kinds = torch.randint(0, 4, (nblk,), generator=g)
    h = torch.where(shape < 2, 16, 32)
    w = torch.where(shape % 2 == 0, 16, 32)
    return h, w, kinds


def c3_block(h: int, w: int, n: int, seed: int, device="cuda") -> torch.Tensor:
    """n blocks of one shape: Laplace(0, 1/sqrt2) innovations (unit variance),
    16*sqrt(2) * L_v Z L_h^T with AR(1) rho = 0.9 (marginal only approx. Laplacian)."""
    g = torch.Generator(device=device).manual_seed(seed)
    u = torch.rand(n, h, w, device=device, generator=g) - 0.5
    # rand() can return exactly 0 (u = -0.5): log1p(-1) = -inf; keep |u| < 0.5
    u = u.clamp_(-0.5 + 2.0 ** -25, 0.5 - 2.0 ** -25)
    z = -(1.0 / math.sqrt(2.0)) * torch.sign(u) * torch.log1p(-2.0 * u.abs())
    lv = ar1_chol(h, 0.9, device, torch.float32)
    lh = ar1_chol(w, 0.9, device, torch.float32)
    return 16.0 * math.sqrt(2.0) * (lv @ z @ lh.T)


C3_SHAPES = ((16, 16), (16, 32), (32, 16), (32, 32))


def c3_fill(x: torch.Tensor, offsets: np.ndarray, first: int, seed: int = 3) -> None:
    """Write blocks [first, first + len(offsets)) of the global config-3 batch
    (shapes from c3_shapes) into the packed buffer x, block i of the range at
    element offsets[i].  Chunk k (CHUNK blocks) draws its blocks of shape s, in
    block order, from seed (seed * 1_000_003 + 4 k + s)."""
    dev = x.device
    offs = torch.from_numpy(np.asarray(offsets, dtype=np.int64)).to(dev)
    gh, gw, _ = _c3_table()
    for k, a, b, d in _chunks(first, len(offsets), CHUNK):
        ch, cw = gh[k * CHUNK:(k + 1) * CHUNK], gw[k * CHUNK:(k + 1) * CHUNK]
        for si, (H, W) in enumerate(C3_SHAPES):
            of_shape = torch.nonzero((ch == H) & (cw == W)).flatten()  # the chunk's draws
            want = (of_shape >= a) & (of_shape < b)
            if not bool(want.any()):
                continue
            blocks = c3_block(H, W, of_shape.numel(), seed=seed * 1_000_003 + 4 * k + si,
                              device=dev)[want.to(dev)]
            local = (of_shape[want] - a + d).to(dev)  # block index within the range
            idx = offs[local][:, None] + torch.arange(H * W, device=dev)[None, :]
            x[idx.flatten()] = blocks.reshape(-1).to(x.dtype)


_C3 = None


def _c3_table():
    global _C3
    if _C3 is None:
        _C3 = c3_shapes(C3_BLOCKS)
    return _C3


def c5_frames(nframes: int = C5_FRAMES, height: int = C5_HEIGHT, width: int = C5_WIDTH,
              device="cuda", offset: int = 0) -> torch.Tensor:
    """Frames [offset, offset + nframes): row-wise then column-wise AR(1) recursion
    x_i = rho x_{i-1} + sqrt(1-rho^2) z_i, x_0 = z_0, scaled by sigma = 30
    (SURVEY.md App. A D12); frame f drawn from seed (5, f)."""
    out = torch.empty(nframes, height, width, device=device, dtype=torch.float32)
    for f in range(nframes):
        g = torch.Generator(device=device).manual_seed(5 * 1_000_003 + offset + f)
        z = torch.randn(height, width, device=device, generator=g)
        rh, rv = 0.92, 0.88
        ch, cv = math.sqrt(1 - rh * rh), math.sqrt(1 - rv * rv)
        # first-order recursive filters as scans: x_i = rho x_{i-1} + c z_i
        x = _ar1_scan(z, rh, ch, dim=1)
        x = _ar1_scan(x, rv, cv, dim=0)
        out[f] = 30.0 * x
    return out


def _ar1_scan(z: torch.Tensor, rho: float, c: float, dim: int) -> torch.Tensor:
    """x_0 = z_0, x_i = rho x_{i-1} + c z_i along `dim`, in log-depth blocks of
    64 (a closed form within each block, a short carry across blocks)."""
    z = z.movedim(dim, -1).double()
    n = z.shape[-1]
    blk = 64
    pad = (-n) % blk
    zz = torch.nn.functional.pad(z, (0, pad))
    m = zz.shape[-1] // blk
    zz = zz.reshape(*zz.shape[:-1], m, blk)
    inc = c * zz
    inc[..., 0, 0] = zz[..., 0, 0]  # x_0 = z_0
    k = torch.arange(blk, device=z.device, dtype=torch.float64)
    # within a block: x_j = sum_{i<=j} rho^(j-i) inc_i  (lower-triangular Toeplitz)
    t = torch.tril(rho ** (k[:, None] - k[None, :]).clamp(min=0))
    t = torch.where(k[:, None] >= k[None, :], t, torch.zeros_like(t))
    local = inc @ t.T
    carry = torch.zeros(*local.shape[:-2], device=z.device, dtype=torch.float64)
    powers = rho ** (k + 1)
    for b in range(m):
        local[..., b, :] += carry[..., None] * powers
        carry = local[..., b, -1]
    x = local.reshape(*local.shape[:-2], m * blk)[..., :n]
    return x.float().movedim(-1, dim)

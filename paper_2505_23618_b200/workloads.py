"""Seeded synthetic inputs for the five BASELINE.json configurations.

No dataset is involved (the paper's VVC test sequences are neither available
nor needed): each config's residuals are generated with the shapes, sizes and
value distributions BASELINE.json states, following SURVEY.md App. A D12-D13.
Generation runs on the GPU with torch (plumbing, outside every timed region)
from torch.Generator(seed); the CPU oracle sees the very same arrays.

  C1  4,096 x 32x32 fp64, separable Gaussian AR(1) rho=0.9, sigma=32, seed 1
  C2  65,536 x 32x32 fp32, AR(1) rho=0.85, sigma=24, rint + clip [-512, 511], seed 2
  C3  1,048,576 blocks, shapes {16,32}^2, Laplace(b=16) innovations mixed by AR(1) 0.9, seed 3
  C4  262,144 x 64x64 fp32, AR(1) rho=0.95, sigma=40, seed 4
  C5  64 frames 3840x2160 fp32, row/column AR(1) recursion rho_h=0.92, rho_v=0.88, sigma=30, seed 5
"""
from __future__ import annotations

import math

import torch


def ar1_chol(n: int, rho: float, device, dtype=torch.float64) -> torch.Tensor:
    i = torch.arange(n, device=device, dtype=torch.float64)
    k = rho ** (i[:, None] - i[None, :]).abs()
    return torch.linalg.cholesky(k).to(dtype)


def ar1_blocks(nblk: int, h: int, w: int, rho: float, sigma: float, seed: int, device="cuda",
               dtype=torch.float32, chunk: int = 1 << 16, offset: int = 0) -> torch.Tensor:
    """sigma * L_v Z L_h^T with Z ~ N(0, 1) i.i.d.  Chunks are seeded
    (seed, chunk index) so a block range is reproducible on any rank."""
    out = torch.empty(nblk, h, w, device=device, dtype=dtype)
    lv = ar1_chol(h, rho, device, torch.float32)
    lh = ar1_chol(w, rho, device, torch.float32)
    for c0 in range(0, nblk, chunk):
        c1 = min(nblk, c0 + chunk)
        g = torch.Generator(device=device).manual_seed(seed * 1_000_003 + (offset + c0) // chunk)
        z = torch.randn(c1 - c0, h, w, device=device, generator=g)
        out[c0:c1] = (sigma * (lv @ z @ lh.T)).to(dtype)
    return out


def c1_inputs(device="cuda", nblk: int = 4096, offset: int = 0) -> torch.Tensor:
    return ar1_blocks(nblk, 32, 32, 0.9, 32.0, 1, device, torch.float64, offset=offset)


def c2_inputs(device="cuda", nblk: int = 65536, offset: int = 0) -> torch.Tensor:
    x = ar1_blocks(nblk, 32, 32, 0.85, 24.0, 2, device, torch.float32, offset=offset)
    return torch.round(x).clamp_(-512, 511)


def c4_inputs(device="cuda", nblk: int = 262144, offset: int = 0) -> torch.Tensor:
    return ar1_blocks(nblk, 64, 64, 0.95, 40.0, 4, device, torch.float32, offset=offset)


def c3_shapes(nblk: int, seed: int = 3) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Per-block (H, W) uniform over {16x16, 16x32, 32x16, 32x32} (H x W read, D9)
    and per-block (h, v) kinds uniform over {DST-7 = 0, DCT-8 = 1}^2 (CPU tensors)."""
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


def c5_frames(nframes: int = 64, height: int = 2160, width: int = 3840, device="cuda",
              offset: int = 0) -> torch.Tensor:
    """Row-wise then column-wise AR(1) recursion x_i = rho x_{i-1} + sqrt(1-rho^2) z_i,
    x_0 = z_0, scaled by sigma = 30."""
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

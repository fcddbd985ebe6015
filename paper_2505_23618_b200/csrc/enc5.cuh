// enc5.cuh -- the simultaneous five-transform encoder evaluation
// (reference pipeline.py:256-293, paper Table 1 "Multiple"): one read of each
// residual block, one shared 2-D DCT-2, five coefficient planes written
//   (dct2,dct2), (dst7,dst7), (dct8,dst7), (dst7,dct8), (dct8,dct8)   [(h, v)]
// where DST-7 / DCT-8 are the DCT-2 plus the 8x8 post-adjustment C7 / C8 = S C7 S
// of each axis.  As in the reference, each DST-7/DCT-8 pair shares one set of
// products (_shared_pair_rows, pipeline.py:242-253): the DCT-8 sums are the
// DST-7 products re-signed, so both planes cost one multiplication set.
// Coefficients outside the first 8 rows / 8 columns are copies of the DCT-2
// plane: bit-identical across the five outputs by construction.
#pragma once
#include "tile_kernel.cuh"

namespace dctadj {

template <typename T>
struct Enc5Params {
  T cv[64];  // vertical C7 (8x8, row-major): mixes coefficient rows 0..7
  T ch[64];  // horizontal C7: mixes coefficient columns 0..7
};

// Phase A, lane per column: R_v[0:8, c] = C_v Y0[0:8, c] for v in {7, 8}
// (8 = chessboard-signed: sum_j s_r s_j C[r][j] y_j, one product set).
// Phase B, lane per row: out(h, v)[r, 0:8] = C_h R_v[r, 0:8] for h in {7, 8}.
template <typename T, int H, int W, int P>
DA_DEV void enc5_stripes(uint8_t* y0, uint8_t* const (&pl)[4], int lane,
                         const Enc5Params<T>& cf) {
  using L = TileLayout<T, H, W, P>;
  // planes: pl[0]=(dst7,dst7) pl[1]=(dct8,dst7) pl[2]=(dst7,dct8) pl[3]=(dct8,dct8)
#pragma unroll 1
  for (int kappa = lane; kappa < P * W; kappa += 32) {
    const uint32_t p = kappa / W, c = kappa % W, byte = c * sizeof(T);
    T y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = *reinterpret_cast<const T*>(y0 + L::addr(p * H + j, byte));
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      T a7 = T(0), a8 = T(0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const T prod = cf.cv[r * 8 + j] * y[j];
        a7 += prod;
        a8 += (j % 2 == 0) ? prod : -prod;
      }
      if (r % 2) a8 = -a8;
      const uint32_t o = L::addr(p * H + r, byte);
      *reinterpret_cast<T*>(pl[0] + o) = a7;
      *reinterpret_cast<T*>(pl[1] + o) = a7;
      *reinterpret_cast<T*>(pl[2] + o) = a8;
      *reinterpret_cast<T*>(pl[3] + o) = a8;
    }
  }
  __syncwarp();
#pragma unroll 1
  for (int rho = lane; rho < P * H; rho += 32) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {  // plane pair (dst7, v) / (dct8, v) shares R_v
      T x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        x[j] = *reinterpret_cast<const T*>(pl[2 * v] + L::addr(rho, j * sizeof(T)));
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        T a7 = T(0), a8 = T(0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const T prod = cf.ch[r * 8 + j] * x[j];
          a7 += prod;
          a8 += (j % 2 == 0) ? prod : -prod;
        }
        if (r % 2) a8 = -a8;
        const uint32_t o = L::addr(rho, r * sizeof(T));
        *reinterpret_cast<T*>(pl[2 * v] + o) = a7;
        *reinterpret_cast<T*>(pl[2 * v + 1] + o) = a8;
      }
    }
  }
}

// One warp per super-tile ring slot (S stages), NG warps per CTA.
template <typename T, int H, int W, int P, int NG, int S>
__global__ void __launch_bounds__(NG * 32)
    enc5_kernel(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap o0,
                const __grid_constant__ CUtensorMap o1, const __grid_constant__ CUtensorMap o2,
                const __grid_constant__ CUtensorMap o3, const __grid_constant__ CUtensorMap o4,
                const __grid_constant__ Geom geom, const __grid_constant__ Enc5Params<T> prm) {
  using L = TileLayout<T, H, W, P>;
  constexpr int RC = op_code(ST_DCT2);
  constexpr int GSQ = H * W;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per warp: S input stages + 4 output planes
  uint8_t* ring = smem + warp * (S + 4) * L::STAGEB;
  uint8_t* const pl[4] = {ring + S * L::STAGEB, ring + (S + 1) * L::STAGEB,
                          ring + (S + 2) * L::STAGEB, ring + (S + 3) * L::STAGEB};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NG * (S + 4) * L::STAGEB) + warp * S;
  const CUtensorMap* outs[5] = {&o0, &o1, &o2, &o3, &o4};
  typename AxisOp<T, W, RC>::Coef nocoef_w;
  typename AxisOp<T, H, RC>::Coef nocoef_h;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * NG + warp;
  const int64_t gstride = static_cast<int64_t>(gridDim.x) * NG;
  const int64_t ntiles = geom.ntiles;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int64_t t = gid + s * gstride;
      if (t < ntiles) {
        mbar_arrive_expect_tx(&bars[s], L::TILEB);
        issue_tile_io<T, H, W, P, MODE_LINEAR>(true, ring + s * L::STAGEB, &in_map, &bars[s], t,
                                               geom, P);
      }
    }
  }
  int s = 0;
  uint32_t phase = 0;
  for (int64_t t = gid, k = 0; t < ntiles; t += gstride, ++k) {
    uint8_t* buf = ring + s * L::STAGEB;
    mbar_wait(&bars[s], phase);
    // the output planes of the previous tile must have been read by its stores
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    row_pass<T, H, W, P, RC, 1, false>(buf, lane, nocoef_w, nullptr);
    __syncwarp();
    col_pass<T, H, W, P, RC, GSQ, false>(buf, lane, nocoef_h, nullptr);
    __syncwarp();
    // copy the DCT-2 plane into the four adjusted planes (same swizzled layout)
    for (int q = lane; q < L::TILEB / 16; q += 32) {
      const uint4 v = reinterpret_cast<const uint4*>(buf)[q];
#pragma unroll
      for (int i = 0; i < 4; ++i) reinterpret_cast<uint4*>(pl[i])[q] = v;
    }
    __syncwarp();
    enc5_stripes<T, H, W, P>(buf, pl, lane, prm);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      issue_tile_io<T, H, W, P, MODE_LINEAR>(false, buf, outs[0], nullptr, t, geom, P);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        issue_tile_io<T, H, W, P, MODE_LINEAR>(false, pl[i], outs[i + 1], nullptr, t, geom, P);
      bulk_commit();
      if (k >= 1) {
        const int64_t tn = t + (S - 1) * gstride;
        if (tn < ntiles) {
          const int sp = (s == 0) ? S - 1 : s - 1;
          bulk_wait_read<1>();
          mbar_arrive_expect_tx(&bars[sp], L::TILEB);
          issue_tile_io<T, H, W, P, MODE_LINEAR>(true, ring + sp * L::STAGEB, &in_map, &bars[sp],
                                                 tn, geom, P);
        }
      }
    }
    __syncwarp();
    if (++s == S) {
      s = 0;
      phase ^= 1;
    }
  }
  if (lane == 0) bulk_wait_all();
}

}  // namespace dctadj

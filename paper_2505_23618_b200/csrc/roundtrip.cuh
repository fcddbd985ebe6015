// roundtrip.cuh -- forward + inverse 2-D adjusted transform of a batch in ONE
// pass over HBM (config 2's step: y = forward(x), x' = inverse(y)).
//
// Per super-tile (P blocks of H x W, TMA-loaded into a ring stage A):
//   forward row pass   (A in place)                     -- reference order: rows,
//   column pass        (A -> registers: forward column op -> y into the group's
//                       staging tile B; inverse column op -> A in place)
//   TMA store B -> y
//   inverse row pass   (A in place)                     -- the inverse's mirror order
//   TMA store A -> x'
// The inverse starts from the forward's fp32/fp64 coefficients in registers,
// which are exactly the values stored to y, and runs the same butterflies in
// the same order as the separate inverse kernel: y and x' are bit-identical to
// dctadj_forward_2d followed by dctadj_inverse_2d.  HBM traffic: x read once,
// y and x' written once (12 B per coefficient pair in fp32 instead of 16 B).
//
// Reference composition: forward_adjusted / inverse_adjusted
// (pipeline.py:176-191) per axis, rows then columns (pipeline.py:236-239).
#pragma once
#include "tile_kernel.cuh"

namespace dctadj {

template <typename T, int W, int H, int RCF, int CCF, int RCI, int CCI>
struct RtParams {
  KParams<T, W, H, RCF, CCF> f;  // forward row / column coefficients
  KParams<T, W, H, RCI, CCI> i;  // inverse row / column coefficients
  T* y;                          // YSTG kernels: coefficients stored from registers
  int64_t nblk;                  // blocks in the batch (the last super-tile may be partial)
};

// Column pass of the round trip: lane owns a column (PAIR: two adjacent columns
// as f2 lanes); forward column op (+ the forward gain removal) -> y tile `yb`,
// then the inverse column op (no scaling: the inverse's last pass is its row
// pass) back into `xb` in place.
// YSTG: y goes straight from registers to HBM (`yg` = the super-tile's first
// block, `nb` blocks of it exist): lane c of the warp stores element (i, c), so
// each store instruction writes whole 128-byte block rows -- no staging tile.
template <typename T, int H, int W, int P, int CCF, int CCI, int GSQF, bool PAIR, bool YSTG,
          int GT = 32>
DA_DEV void col_pass_rt(uint8_t* xb, uint8_t* yb, T* yg, int nb, int lane,
                        const typename AxisOp<T, H, CCF>::Coef& cff,
                        const typename AxisOp<T, H, CCI>::Coef& cfi) {
  using L = TileLayout<T, H, W, P>;
  constexpr int COLS_PER_IT = PAIR ? 2 * GT : GT;
  static_assert((P * W) % COLS_PER_IT == 0, "column pass must cover whole warps");
#pragma unroll 1
  for (int it = 0; it < (P * W) / COLS_PER_IT; ++it) {
    const int kappa = it * COLS_PER_IT + (PAIR ? 2 : 1) * lane;
    const uint32_t p = kappa / W, c = kappa % W;
    const uint32_t byte = c * sizeof(T);
    if constexpr (!PAIR) {
      T v[H];
#pragma unroll
      for (int i = 0; i < H; ++i) v[i] = *reinterpret_cast<const T*>(xb + L::addr(p * H + i, byte));
      apply_axis<T, H, CCF>(v, cff, nullptr);
      scale_out<T, H, GSQF>(v);
      if constexpr (YSTG) {
        if (static_cast<int>(p) < nb) {
          T* dst = yg + static_cast<size_t>(p) * H * W + c;
#pragma unroll
          for (int i = 0; i < H; ++i) __stcs(dst + i * W, v[i]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < H; ++i) *reinterpret_cast<T*>(yb + L::addr(p * H + i, byte)) = v[i];
      }
      apply_axis<T, H, CCI>(v, cfi, nullptr);
#pragma unroll
      for (int i = 0; i < H; ++i) *reinterpret_cast<T*>(xb + L::addr(p * H + i, byte)) = v[i];
    } else {
      static_assert(sizeof(T) == 4, "packed columns are fp32 pairs");
      f2 v[H];
#pragma unroll
      for (int i = 0; i < H; ++i)
        v[i].v = *reinterpret_cast<const float2*>(xb + L::addr(p * H + i, byte));
      apply_axis<f2, H, CCF>(v, cff, nullptr);
      scale_out<f2, H, GSQF>(v);
      if constexpr (YSTG) {
        if (static_cast<int>(p) < nb) {
          float2* dst = reinterpret_cast<float2*>(yg + static_cast<size_t>(p) * H * W + c);
#pragma unroll
          for (int i = 0; i < H; ++i) __stcs(dst + i * (W / 2), v[i].v);
        }
      } else {
#pragma unroll
        for (int i = 0; i < H; ++i)
          *reinterpret_cast<float2*>(yb + L::addr(p * H + i, byte)) = v[i].v;
      }
      apply_axis<f2, H, CCI>(v, cfi, nullptr);
#pragma unroll
      for (int i = 0; i < H; ++i) *reinterpret_cast<float2*>(xb + L::addr(p * H + i, byte)) = v[i].v;
    }
  }
}

// NG groups of NW warps per CTA; each group owns an S-stage ring of input
// super-tiles and one y staging tile (NW > 1: a tile's rows / columns are split
// across the group's warps, which meet at a named barrier).  Persistent grid,
// static stride over super-tiles (blocks are independent), programmatic
// dependent launch like the tile kernel.
template <typename T, int H, int W, int P, int RCF, int CCF, int RCI, int CCI, int NG, int S,
          bool PAIR_ROW_F, bool PAIR_COL, bool PAIR_ROW_I, int MINB, bool YSTG, int NW = 1,
          int CH = 0,  // CH: L2 hints, 1 = loads evict_first, 2 = stores evict_first
          int MODE = MODE_LINEAR>
__global__ void __launch_bounds__(NG * NW * 32, MINB)
    roundtrip_kernel(const __grid_constant__ CUtensorMap in_map,
                     const __grid_constant__ CUtensorMap y_map,
                     const __grid_constant__ CUtensorMap xr_map, const __grid_constant__ Geom geom,
                     const __grid_constant__ RtParams<T, W, H, RCF, CCF, RCI, CCI> prm) {
  using L = TileLayout<T, H, W, P>;
  using RowF = AxisOp<T, W, RCF>;
  using ColF = AxisOp<T, H, CCF>;
  using RowI = AxisOp<T, W, RCI>;
  using ColI = AxisOp<T, H, CCI>;
  static_assert(!RowF::kDense && !ColF::kDense && !RowI::kDense && !ColI::kDense,
                "the round trip fuses the fast paths");
  static_assert(!RowF::kIdentity && !ColF::kIdentity && !RowI::kIdentity && !ColI::kIdentity,
                "2-D round trip: every pass has an op");
  static_assert(S >= 2, "ring needs at least two stages");
  constexpr int GSQF = RowF::kGainSq * ColF::kGainSq;
  constexpr int GSQI = RowI::kGainSq * ColI::kGainSq;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  if (!geom.early) asm volatile("griddepcontrol.wait;" ::: "memory");  // see Geom::early
  asm volatile("griddepcontrol.launch_dependents;" :::);
  constexpr int GT = NW * 32;
  static_assert(NW == 1 || NG <= 15, "named barriers 1..15");
  const int grp = threadIdx.x / GT, lane = threadIdx.x % GT;
  constexpr int NBUF = YSTG ? S : S + 1;  // ring stages (+ the y staging tile)
  uint8_t* ring = smem + grp * NBUF * L::STAGEB;
  uint8_t* ybuf = ring + S * L::STAGEB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NG * NBUF * L::STAGEB) + grp * S;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    if (grp == 0) {
      prefetch_map(&in_map);
      prefetch_map(&y_map);
      prefetch_map(&xr_map);
    }
  }
  group_sync<NW>(grp);

  const int64_t gid = static_cast<int64_t>(blockIdx.x) * NG + grp;
  const int64_t gstride = static_cast<int64_t>(gridDim.x) * NG;
  const int64_t ntiles = geom.ntiles;
  // GATHER (config 3): one TMA box per block at its element offset in a packed
  // mixed-shape buffer; lane p < P moves block p of every super-tile (loads and
  // both stores), so each lane's bulk-group accounting covers its own block.
  // The offsets of the tiles in flight are kept per stage, the next refill's
  // prefetched into a register.
  constexpr bool GATHER = MODE == MODE_GATHER;
  static_assert(MODE == MODE_LINEAR || MODE == MODE_GATHER, "linear or gather batches");
  static_assert(!GATHER || (!YSTG && P <= GT), "gather: staged y, one lane per block");
  __shared__ int64_t goffs[GATHER ? NG * S * P : 1];
  int64_t* my_offs = goffs + (GATHER ? grp * S * P : 0);
  int64_t pref = 0;
  auto load = [&](int st, int64_t t, int64_t off) {  // GATHER: every lane; else lane 0
    const int nb = tile_blocks<P, MODE>(t, geom);
    if constexpr (GATHER) {
      if (lane == 0) mbar_arrive_expect_tx(&bars[st], L::TILEB / P * nb);
      group_sync<NW>(grp);
      if (lane < P) my_offs[st * P + lane] = off;
      gather_io<T, H, W, P>(true, ring + st * L::STAGEB, &in_map, &bars[st], lane, nb, off);
    } else {
      mbar_arrive_expect_tx(&bars[st], L::TILEB);
      issue_tile_io<T, H, W, P, MODE_LINEAR, CH>(true, ring + st * L::STAGEB, &in_map, &bars[st],
                                                 t, geom, P);
    }
  };
  auto store = [&](const CUtensorMap* map, uint8_t* src, int st, int64_t t) {
    if constexpr (GATHER) {
      gather_io<T, H, W, P>(false, src, map, nullptr, lane, tile_blocks<P, MODE>(t, geom),
                            lane < P ? my_offs[st * P + lane] : 0);
      bulk_commit();
    } else if (lane == 0) {
      issue_tile_io<T, H, W, P, MODE_LINEAR, CH>(false, src, map, nullptr, t, geom, P);
      bulk_commit();
    }
  };
  auto offset_of = [&](int64_t t) -> int64_t {  // GATHER: this lane's block of tile t
    if constexpr (GATHER)
      return (t < ntiles && lane < tile_blocks<P, MODE>(t, geom)) ? geom.offsets[t * P + lane] : 0;
    else
      return 0;
  };
#pragma unroll
  for (int st = 0; st < S; ++st) {
    const int64_t t = gid + st * gstride;
    if (t < ntiles && (GATHER || lane == 0)) load(st, t, offset_of(t));
  }
  if constexpr (GATHER) pref = offset_of(gid + S * gstride);

  int s = 0;
  uint32_t phase = 0;
  for (int64_t t = gid, k = 0; t < ntiles; t += gstride, ++k) {
    uint8_t* buf = ring + s * L::STAGEB;
    mbar_wait(&bars[s], phase);
    row_pass<T, H, W, P, RCF, 1, PAIR_ROW_F, GT>(buf, lane, prm.f.row, nullptr);
    if constexpr (!YSTG) {
      // y of the previous tile must have left the staging tile (groups pending
      // at this point: y(k-1), x'(k-1))
      if (GATHER || lane == 0) bulk_wait_read<1>();
    }
    group_sync<NW>(grp);
    const int64_t left = prm.nblk - t * P;
    col_pass_rt<T, H, W, P, CCF, CCI, GSQF, PAIR_COL, YSTG, GT>(
        buf, ybuf, prm.y + static_cast<size_t>(t) * P * H * W, left < P ? static_cast<int>(left) : P,
        lane, prm.f.col, prm.i.col);
    if constexpr (!YSTG) {
      fence_proxy_async_smem();
      group_sync<NW>(grp);
      store(&y_map, ybuf, s, t);
    }
    if constexpr (YSTG) group_sync<NW>(grp);  // the column pass is complete
    row_pass<T, H, W, P, RCI, GSQI, PAIR_ROW_I, GT>(buf, lane, prm.i.row, nullptr);
    fence_proxy_async_smem();
    group_sync<NW>(grp);
    store(&xr_map, buf, s, t);
    // refill the stage of the previous tile with the tile S-1 strides ahead,
    // once its x' store has read it (pending after that: [y(k),] x'(k))
    if (k >= 1) {
      const int64_t tn = t + (S - 1) * gstride;
      if (tn < ntiles && (GATHER || lane == 0)) {
        const int sp = (s == 0) ? S - 1 : s - 1;
        bulk_wait_read<YSTG ? 1 : 2>();
        load(sp, tn, pref);
        if constexpr (GATHER) pref = offset_of(tn + gstride);
      }
    }
    group_sync<NW>(grp);
    if (++s == S) {
      s = 0;
      phase ^= 1;
    }
  }
  if (GATHER || lane == 0) bulk_wait_all();
  if (geom.early) asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace dctadj

// ------------------------------------------------------------------ host side
namespace dctadj {

struct RtArgs {
  const void* in = nullptr;  // x   (rows x W, LINEAR)
  void* y = nullptr;         // y   (forward coefficients)
  void* xr = nullptr;        // x'  (reconstruction)
  int64_t rows = 0;          // LINEAR: nblk * H; GATHER: rows of W in the packed buffer
  const void* coef[4] = {};  // host, packed Coef of: forward row, forward column, inverse row, inverse column
  const int64_t* offsets = nullptr;  // GATHER: device, element offset of each block
  int64_t gather_blocks = 0;         // GATHER: blocks of this class
  cudaStream_t stream = nullptr;
};

struct RtEntry {
  int dtype, h, w, rcf, ccf, rci, cci, mode, variant;
  int (*fn)(const RtArgs&);
};

// implemented in roundtrip.cu: the fused kernel for these ops and addressing
// mode (MODE_LINEAR / MODE_GATHER), or nullptr
const RtEntry* find_roundtrip(int dtype, int h, int w, int rcf, int ccf, int rci, int cci,
                              int mode, int variant);

}  // namespace dctadj

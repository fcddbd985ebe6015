// tile_kernel.cuh -- the one persistent, TMA-fed tile kernel behind every
// entry point of the C-ABI.
//
// A "super-tile" is P consecutive H x W blocks (P*H rows of W samples).  Each
// warp owns an S-stage ring of super-tile buffers in shared memory:
//   TMA 2-D tile load (128B/64B/32B swizzle, zero-filled out of bounds)
//     -> mbarrier complete_tx
//     -> row pass: lane r owns row r, 16-byte swizzled LDS into registers,
//        register butterfly + adjustment, STS back in place
//     -> column pass: lane c owns column c (conflict-free under the swizzle)
//     -> fence.proxy.async -> TMA 2-D tile store (clipped out of bounds)
// The forward transform runs rows then columns (reference pipeline.py:236-239);
// the inverse runs columns then rows (its mirror).  The 1-D batch API is the
// same kernel with 32 vectors per tile and no column op.
//
// Blocks are independent (reference SPEC.md:313-314), so warps walk the tile
// list with a static grid stride; HBM traffic is one read and one write per
// sample.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "butterfly.cuh"

namespace dctadj {

// ---------------------------------------------------------------- PTX helpers
DA_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
DA_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
DA_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
DA_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
DA_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
DA_DEV bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
DA_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "DA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra DA_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
DA_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
DA_DEV void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                        int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
DA_DEV void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
DA_DEV void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                        int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
DA_DEV void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
DA_DEV void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// L2 eviction-priority hints for streaming data (read once / written once)
DA_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
DA_DEV void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
DA_DEV void tma_store_2d_hint(const CUtensorMap* map, const void* src, int c0, int c1,
                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint"
      " [%0, {%2, %3}], [%1], %4;" ::"l"(map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
DA_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
DA_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
DA_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
DA_DEV void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
DA_DEV void prefetch_map(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}

// ------------------------------------------------------------------ layout
// Row bytes W*sizeof(T) are cut into boxes of BRB = min(row bytes, 128) bytes;
// box b of the super-tile occupies BOXB = P*H*BRB contiguous smem bytes with the
// matching TMA swizzle (128B/64B/32B; none for 16-byte rows).
template <typename T, int H, int W, int P>
struct TileLayout {
  static constexpr int ES = sizeof(T);
  static constexpr int ROWB = W * ES;
  static constexpr int BRB = ROWB < 128 ? ROWB : 128;
  static constexpr int NB = ROWB / BRB;
  static constexpr int BW = BRB / ES;  // elements per box row
  static constexpr int PH = P * H;
  static constexpr int BOXB = PH * BRB;
  static constexpr int TILEB = NB * BOXB;
  static constexpr int STAGEB = (TILEB + 1023) / 1024 * 1024;
  static constexpr int SWZ_MASK = BRB == 128 ? 7 : BRB == 64 ? 3 : BRB == 32 ? 1 : 0;
  static_assert(BRB >= 16, "rows shorter than 16 bytes are not TMA-addressable");
  static_assert(PH % 32 == 0, "super-tile rows must cover whole warps");
  // physical byte offset of (row rho, byte offset `byte` within the row)
  static DA_DEV uint32_t addr(uint32_t rho, uint32_t byte) {
    const uint32_t b = byte / BRB, off = byte % BRB;
    const uint32_t a = rho * BRB + off;
    return b * BOXB + (a ^ (((a >> 7) & SWZ_MASK) << 4));
  }
  // Column walks: rows rho0 + i * STEP at one byte offset.  The swizzle term of
  // every TMA pattern above repeats every 8 rows, so addr(rho0 + i STEP, byte) =
  // base[i % M] + i * STEP * BRB with M = 8 / gcd(STEP, 8): a per-lane base
  // register plus an immediate, no integer work per element once i is unrolled.
  template <int STEP>
  struct Col {
    static constexpr int M = 8 / (STEP % 8 == 0 ? 8 : STEP % 4 == 0 ? 4 : STEP % 2 == 0 ? 2 : 1);
    uint32_t base[M];
    DA_DEV Col(uint32_t rho0, uint32_t byte) {
#pragma unroll
      for (int m = 0; m < M; ++m) base[m] = addr(rho0 + m * STEP, byte) - m * STEP * BRB;
    }
    DA_DEV uint32_t operator()(int i) const { return base[i % M] + i * STEP * BRB; }
  };
};

// LINEAR: super-tile t = rows [t*P*H, (t+1)*P*H) of a [rows, W] view.
// FRAME:  blocks in raster order of (F, height, width) frames.
// GATHER: block i of a class list sits at element offset offsets[i] of a packed
//         mixed-shape buffer viewed as [elements / W, W] (config 3).
// MODE_FRAME4 (tensor-core dense kernel only): a super-tile of 4 horizontally
// adjacent blocks moves as ONE 4-D box {32 cols, 4 blocks, 32 rows, 1 frame}, so
// each frame row is a single 512-byte segment; the smem tile is then row-
// interleaved (tile row = 4 * block row + block) instead of block-major.
//
// MODE_FRAME_IL / MODE_LINEAR_IL (tile kernel, rows of <= 128 bytes): the same
// idea for a P-block super-tile -- the frame side is one 4-D box {W, P blocks,
// H rows, 1}, the block-major side one 3-D box {W, P blocks, H rows} over
// (nblk, H, W) -- and both sides see the row-interleaved smem tile.
enum Mode : int {
  MODE_LINEAR = 0,
  MODE_FRAME = 1,
  MODE_GATHER = 2,
  MODE_FRAME4 = 3,
  MODE_FRAME_IL = 4,
  MODE_LINEAR_IL = 5
};
template <int MODE>
__host__ __device__ constexpr bool is_il_mode() {
  return MODE == MODE_FRAME_IL || MODE == MODE_LINEAR_IL;
}

struct Geom {
  int64_t ntiles;      // super-tiles
  int64_t nblocks;     // blocks (FRAME: a super-tile holds P consecutive raster blocks)
  int32_t tiles_y;     // FRAME: tile rows per frame
  int32_t tiles_x;     // FRAME: tile columns per frame
  const void* dense_row;  // device N x N (T) for ST_DENSE row op
  const void* dense_col;  // device N x N (T) for ST_DENSE column op
  const int64_t* offsets; // GATHER: element offset of each block (device)
  int32_t early;          // 1: independent of every launch still in flight on the stream
                          // (host-checked, pdl_early): skip the entry griddepcontrol.wait
                          // and wait at exit instead, so this grid's loads and passes
                          // overlap the previous grid's tail but it never completes first
};

template <typename T, int W, int H, int RC, int CC>
struct KParams {
  typename AxisOp<T, W, RC>::Coef row;
  typename AxisOp<T, H, CC>::Coef col;
};

// GATHER: lane p < nb moves block p of the super-tile (element offset `off`).
template <typename T, int H, int W, int P>
DA_DEV void gather_io(bool load, void* stage, const CUtensorMap* map, uint64_t* bar, int lane,
                      int nb, int64_t off) {
  using L = TileLayout<T, H, W, P>;
  if (lane >= nb) return;
  const int row0 = static_cast<int>(off / W);
#pragma unroll
  for (int b = 0; b < L::NB; ++b) {
    uint8_t* d = static_cast<uint8_t*>(stage) + b * L::BOXB + lane * H * L::BRB;
    if (load)
      tma_load_2d(d, map, bar, b * L::BW, row0);
    else
      tma_store_2d(map, d, b * L::BW, row0);
  }
}

// Blocks of super-tile t that exist (a FRAME super-tile may be cut short).
template <int P, int MODE>
DA_DEV int tile_blocks(int64_t t, const Geom& g) {
  if constexpr (MODE == MODE_LINEAR || is_il_mode<MODE>()) {
    return P;
  } else {
    const int64_t left = g.nblocks - t * P;
    return left < P ? static_cast<int>(left) : P;
  }
}

// TMA loads (load=true) or stores of super-tile t.  LINEAR: one box per
// 128-byte column slice covering all P*H rows.  FRAME: one box per block and
// column slice, block b -> (frame, tile row, tile column) in raster order.
// CH: L2 hint bits -- 1: loads evict_first, 2: stores evict_first
template <typename T, int H, int W, int P, int MODE, int CH = 0>
DA_DEV void issue_tile_io(bool load, void* stage, const CUtensorMap* map, uint64_t* bar,
                          int64_t t, const Geom& g, int nb) {
  using L = TileLayout<T, H, W, P>;
  if constexpr (is_il_mode<MODE>()) {
    static_assert(L::NB == 1, "interleaved tiles need rows of <= 128 bytes");
    if constexpr (MODE == MODE_LINEAR_IL) {
      const int b0 = static_cast<int>(t * P);
      if (load)
        tma_load_3d(stage, map, bar, 0, b0, 0);
      else
        tma_store_3d(map, stage, 0, b0, 0);
    } else {
      const int64_t per = static_cast<int64_t>(g.tiles_x) * g.tiles_y, blk = t * P;
      const int f = static_cast<int>(blk / per);
      const int rem = static_cast<int>(blk - f * per);
      const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
      if (load)
        tma_load_4d(stage, map, bar, 0, tx, ty * H, f);
      else
        tma_store_4d(map, stage, 0, tx, ty * H, f);
    }
    return;
  }
#pragma unroll
  for (int b = 0; b < L::NB; ++b) {
    uint8_t* dst = static_cast<uint8_t*>(stage) + b * L::BOXB;
    if constexpr (MODE == MODE_LINEAR) {
      const int row0 = static_cast<int>(t * L::PH);
      if (load) {
        if constexpr (CH & 1)
          tma_load_2d_hint(dst, map, bar, b * L::BW, row0, policy_evict_first());
        else
          tma_load_2d(dst, map, bar, b * L::BW, row0);
      } else {
        if constexpr (CH & 2)
          tma_store_2d_hint(map, dst, b * L::BW, row0, policy_evict_first());
        else
          tma_store_2d(map, dst, b * L::BW, row0);
      }
    } else {
      const int64_t per = static_cast<int64_t>(g.tiles_x) * g.tiles_y;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (p >= nb) break;
        const int64_t blk = t * P + p;
        const int f = static_cast<int>(blk / per);
        const int rem = static_cast<int>(blk - f * per);
        const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
        uint8_t* d = dst + p * H * L::BRB;
        if (load)
          tma_load_3d(d, map, bar, tx * W + b * L::BW, ty * H, f);
        else
          tma_store_3d(map, d, tx * W + b * L::BW, ty * H, f);
      }
    }
  }
}

// 1 / (gain_row * gain_col), gains^2 being powers of two: exact unless odd exponent
__host__ __device__ constexpr double inv_sqrt_pow2(int gsq) {
  int e = 0;
  while ((1 << e) < gsq) ++e;
  double s = 1.0;
  for (int i = 0; i < e / 2; ++i) s *= 0.5;
  return (e % 2) ? s * K_SQRT1_2 : s;
}

template <typename V, int N, int GSQ>
DA_DEV void scale_out(V (&v)[N]) {
  if constexpr (GSQ > 1) {
    using Sc = typename Scalar<V>::type;
    constexpr Sc sc = Sc(inv_sqrt_pow2(GSQ));
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = mul(v[i], sc);
  }
}

// Row pass: lane owns a row (PAIR: two rows, rho and rho + GT, packed as f2
// lanes).  Rows are read/written as 16-byte chunks: conflict-free under the
// swizzle (8 lanes of a phase hit 8 distinct chunk columns).
//
// row_pass_io reads the tile from `in` and writes the result to `out` (same
// layout; in == out is the in-place pass).
template <typename T, int H, int W, int P, int RC, int GSQ, bool PAIR, int GT = 32>
DA_DEV void row_pass_io(const uint8_t* in, uint8_t* out, int lane,
                        const typename AxisOp<T, W, RC>::Coef& cf, const T* dense) {
  using L = TileLayout<T, H, W, P>;
  constexpr int PER16 = 16 / sizeof(T);
  constexpr int ROWS_PER_IT = PAIR ? 2 * GT : GT;
  static_assert(L::PH % ROWS_PER_IT == 0, "row pass must cover whole warps");
#pragma unroll 1
  for (int it = 0; it < L::PH / ROWS_PER_IT; ++it) {
    const uint32_t rho = it * ROWS_PER_IT + lane;
    if constexpr (!PAIR) {
      T v[W];
#pragma unroll
      for (int q = 0; q < W / PER16; ++q) {
        const uint4 raw = *reinterpret_cast<const uint4*>(in + L::addr(rho, q * 16));
        const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int k = 0; k < PER16; ++k) v[q * PER16 + k] = e[k];
      }
      apply_axis<T, W, RC>(v, cf, dense);
      scale_out<T, W, GSQ>(v);
#pragma unroll
      for (int q = 0; q < W / PER16; ++q) {
        uint4 raw;
        T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
        for (int k = 0; k < PER16; ++k) e[k] = v[q * PER16 + k];
        *reinterpret_cast<uint4*>(out + L::addr(rho, q * 16)) = raw;
      }
    } else {
      static_assert(sizeof(T) == 4, "packed rows are fp32 pairs");
      f2 v[W];
#pragma unroll
      for (int q = 0; q < W / 4; ++q) {
        const float4 a = *reinterpret_cast<const float4*>(in + L::addr(rho, q * 16));
        const float4 b = *reinterpret_cast<const float4*>(in + L::addr(rho + GT, q * 16));
        v[4 * q + 0].v = make_float2(a.x, b.x);
        v[4 * q + 1].v = make_float2(a.y, b.y);
        v[4 * q + 2].v = make_float2(a.z, b.z);
        v[4 * q + 3].v = make_float2(a.w, b.w);
      }
      apply_axis<f2, W, RC>(v, cf, dense);
      scale_out<f2, W, GSQ>(v);
#pragma unroll
      for (int q = 0; q < W / 4; ++q) {
        *reinterpret_cast<float4*>(out + L::addr(rho, q * 16)) =
            make_float4(v[4 * q].v.x, v[4 * q + 1].v.x, v[4 * q + 2].v.x, v[4 * q + 3].v.x);
        *reinterpret_cast<float4*>(out + L::addr(rho + GT, q * 16)) =
            make_float4(v[4 * q].v.y, v[4 * q + 1].v.y, v[4 * q + 2].v.y, v[4 * q + 3].v.y);
      }
    }
  }
}

template <typename T, int H, int W, int P, int RC, int GSQ, bool PAIR, int GT = 32>
DA_DEV void row_pass(uint8_t* buf, int lane, const typename AxisOp<T, W, RC>::Coef& cf,
                     const T* dense) {
  row_pass_io<T, H, W, P, RC, GSQ, PAIR, GT>(buf, buf, lane, cf, dense);
}

// Column pass: lane owns a column (PAIR: two adjacent columns read as one
// 8-byte word, packed as f2 lanes).  Conflict-free under the swizzle.
// COLADDR: walk the column with TileLayout::Col's precomputed bases (a register
// plus an immediate per element) instead of recomputing each swizzled address --
// fewer integer instructions, which pays in the issue-bound fused config-5
// kernel; measured neutral (block-major) to 6 % slower (interleaved frame
// kernels) in the tile kernels, which keep the per-element form.
template <typename T, int H, int W, int P, int CC, int GSQ, bool PAIR, int GT = 32,
          bool IL = false, bool COLADDR = false>
DA_DEV void col_pass(uint8_t* buf, int lane, const typename AxisOp<T, H, CC>::Coef& cf,
                     const T* dense) {
  using L = TileLayout<T, H, W, P>;
  // tile row of (block p, block row i): block-major, or row-interleaved (IL)
  constexpr int COLS_PER_IT = PAIR ? 2 * GT : GT;
  static_assert((P * W) % COLS_PER_IT == 0, "column pass must cover whole warps");
#pragma unroll 1
  for (int it = 0; it < (P * W) / COLS_PER_IT; ++it) {
    const int kappa = it * COLS_PER_IT + (PAIR ? 2 : 1) * lane;
    const uint32_t p = kappa / W, c = kappa % W;
    // tile row of (block p, block row i): block-major, or row-interleaved (IL)
    const typename L::template Col<IL ? P : 1> col(IL ? p : p * H, c * sizeof(T));
    auto at = [&](int i) -> uint32_t {
      return COLADDR ? col(i) : L::addr(IL ? i * P + p : p * H + i, c * sizeof(T));
    };
    if constexpr (!PAIR) {
      T v[H];
#pragma unroll
      for (int i = 0; i < H; ++i) v[i] = *reinterpret_cast<const T*>(buf + at(i));
      apply_axis<T, H, CC>(v, cf, dense);
      scale_out<T, H, GSQ>(v);
#pragma unroll
      for (int i = 0; i < H; ++i) *reinterpret_cast<T*>(buf + at(i)) = v[i];
    } else {
      static_assert(sizeof(T) == 4, "packed columns are fp32 pairs");
      f2 v[H];
#pragma unroll
      for (int i = 0; i < H; ++i) v[i].v = *reinterpret_cast<const float2*>(buf + at(i));
      apply_axis<f2, H, CC>(v, cf, dense);
      scale_out<f2, H, GSQ>(v);
#pragma unroll
      for (int i = 0; i < H; ++i) *reinterpret_cast<float2*>(buf + at(i)) = v[i].v;
    }
  }
}

// NG groups of NW warps per CTA; each group owns an S-stage ring and works one
// super-tile at a time (NW > 1: the rows / columns of a tile are split across
// the group's warps, synchronised by a named barrier).
template <int NW>
DA_DEV void group_sync(int grp) {
  if constexpr (NW == 1)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "n"(NW * 32) : "memory");
}

template <typename T, int H, int W, int P, int RC, int CC, bool COL_FIRST, int IN_MODE,
          int OUT_MODE, int NG, int S, bool PAIR_ROW = false, bool PAIR_COL = false, int CH = 0,
          int NW = 1>
// CH bits 0-1: L2 hints; bit 3: the launcher runs ring_kernel instead (below);
// bits 4+: minimum resident CTAs per SM (register cap)
__global__ void __launch_bounds__(NG * NW * 32, (CH >> 4) > 0 ? (CH >> 4) : 1)
    tile_kernel(const __grid_constant__ CUtensorMap in_map,
                const __grid_constant__ CUtensorMap out_map, const __grid_constant__ Geom geom,
                const __grid_constant__ KParams<T, W, H, RC, CC> prm) {
  using L = TileLayout<T, H, W, P>;
  using RowOp = AxisOp<T, W, RC>;
  using ColOp = AxisOp<T, H, CC>;
  constexpr int GT = NW * 32;
  static_assert(NG * NW <= 32 && (NW == 1 || NG <= 15), "named barriers 1..15");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // dynamic smem is only guaranteed 16-byte aligned: round up to 1024 for the swizzle atom
  // (pointer arithmetic, not an integer round trip, keeps the shared address space)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // Programmatic dependent launch: this grid may have been scheduled while the
  // previous kernel in the stream drains; wait for it before touching memory
  // (unless the host proved the two independent: geom.early), and let the next
  // kernel get scheduled as our CTAs retire.
  if (!geom.early) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  // `lane`: thread index within the group (0 .. NW*32-1)
  const int grp = threadIdx.x / GT, lane = threadIdx.x % GT;
  uint8_t* ring = smem + grp * S * L::STAGEB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NG * S * L::STAGEB) + grp * S;
  T* dense_base = reinterpret_cast<T*>(smem + NG * S * L::STAGEB + NG * S * 8);
  T* dense_row = dense_base;
  T* dense_col = dense_base + (RowOp::kDense ? W * W : 0);

  if constexpr (RowOp::kDense || ColOp::kDense) {
    if constexpr (RowOp::kDense) {
      const T* src = static_cast<const T*>(geom.dense_row);
      for (int i = threadIdx.x; i < W * W; i += NG * GT) dense_row[i] = src[i];
    }
    if constexpr (ColOp::kDense) {
      const T* src = static_cast<const T*>(geom.dense_col);
      for (int i = threadIdx.x; i < H * H; i += NG * GT) dense_col[i] = src[i];
    }
    __syncthreads();
  }

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    if (grp == 0) {
      prefetch_map(&in_map);
      prefetch_map(&out_map);
    }
  }
  group_sync<NW>(grp);

  const int64_t gid = static_cast<int64_t>(blockIdx.x) * NG + grp;
  const int64_t gstride = static_cast<int64_t>(gridDim.x) * NG;
  const int64_t ntiles = geom.ntiles;

  constexpr bool GATHER = IN_MODE == MODE_GATHER;
  static_assert(GATHER == (OUT_MODE == MODE_GATHER), "gather mode is in+out");
  constexpr bool IL = is_il_mode<IN_MODE>();
  static_assert(IL == is_il_mode<OUT_MODE>(), "interleaved tiles are in+out");
  static_assert(!GATHER || P <= GT, "one thread per gathered block");
  // GATHER: the offsets of the blocks in flight (stage-major) and a register
  // prefetch of the next refill's offsets, one lane per block
  __shared__ int64_t goffs[GATHER ? NG * S * P : 1];
  int64_t* my_offs = goffs + (GATHER ? grp * S * P : 0);
  int64_t pref = 0;

  if constexpr (!GATHER) {
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int64_t t = gid + s * gstride;
        if (t < ntiles) {
          const int nb = tile_blocks<P, IN_MODE>(t, geom);
          mbar_arrive_expect_tx(&bars[s], L::TILEB / P * nb);
          issue_tile_io<T, H, W, P, IN_MODE, CH>(true, ring + s * L::STAGEB, &in_map, &bars[s], t,
                                                 geom, nb);
        }
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int64_t t = gid + s * gstride;
      if (t < ntiles) {
        const int nb = tile_blocks<P, IN_MODE>(t, geom);
        if (lane == 0) mbar_arrive_expect_tx(&bars[s], L::TILEB / P * nb);
        group_sync<NW>(grp);
        const int64_t off = lane < nb ? geom.offsets[t * P + lane] : 0;
        if (lane < P) my_offs[s * P + lane] = off;
        gather_io<T, H, W, P>(true, ring + s * L::STAGEB, &in_map, &bars[s], lane, nb, off);
      }
    }
    const int64_t tp = gid + S * gstride;
    if (tp < ntiles && lane < tile_blocks<P, IN_MODE>(tp, geom)) pref = geom.offsets[tp * P + lane];
  }

  int s = 0;
  uint32_t phase = 0;
  for (int64_t t = gid, k = 0; t < ntiles; t += gstride, ++k) {
    uint8_t* buf = ring + s * L::STAGEB;
    mbar_wait(&bars[s], phase);
    // the unnormalized base gains of both axes are removed in the last pass
    constexpr int GSQ = RowOp::kGainSq * ColOp::kGainSq;
    if constexpr (!COL_FIRST) {
      if constexpr (!RowOp::kIdentity) {
        row_pass<T, H, W, P, RC, ColOp::kIdentity ? GSQ : 1, PAIR_ROW, GT>(buf, lane, prm.row,
                                                                          dense_row);
        if constexpr (!ColOp::kIdentity) group_sync<NW>(grp);
      }
      if constexpr (!ColOp::kIdentity)
        col_pass<T, H, W, P, CC, GSQ, PAIR_COL, GT, IL>(buf, lane, prm.col, dense_col);
    } else {
      if constexpr (!ColOp::kIdentity) {
        col_pass<T, H, W, P, CC, RowOp::kIdentity ? GSQ : 1, PAIR_COL, GT, IL>(buf, lane, prm.col,
                                                                              dense_col);
        if constexpr (!RowOp::kIdentity) group_sync<NW>(grp);
      }
      if constexpr (!RowOp::kIdentity)
        row_pass<T, H, W, P, RC, GSQ, PAIR_ROW, GT>(buf, lane, prm.row, dense_row);
    }
    fence_proxy_async_smem();
    group_sync<NW>(grp);
    if constexpr (!GATHER) {
      if (lane == 0) {
        issue_tile_io<T, H, W, P, OUT_MODE, CH>(false, buf, &out_map, nullptr, t, geom,
                                                tile_blocks<P, OUT_MODE>(t, geom));
        bulk_commit();
        // refill the stage freed by the previous tile with the tile S-1 strides ahead
        if (k >= 1) {
          const int64_t tn = t + (S - 1) * gstride;
          if (tn < ntiles) {
            const int sp = (s == 0) ? S - 1 : s - 1;
            bulk_wait_read<1>();
            const int nb = tile_blocks<P, IN_MODE>(tn, geom);
            mbar_arrive_expect_tx(&bars[sp], L::TILEB / P * nb);
            issue_tile_io<T, H, W, P, IN_MODE, CH>(true, ring + sp * L::STAGEB, &in_map, &bars[sp],
                                                   tn, geom, nb);
          }
        }
      }
    } else {
      const int nbt = tile_blocks<P, OUT_MODE>(t, geom);
      gather_io<T, H, W, P>(false, buf, &out_map, nullptr, lane, nbt,
                            lane < P ? my_offs[s * P + lane] : 0);
      bulk_commit();
      if (k >= 1) {
        const int64_t tn = t + (S - 1) * gstride;
        if (tn < ntiles) {
          const int sp = (s == 0) ? S - 1 : s - 1;
          bulk_wait_read<1>();
          const int nb = tile_blocks<P, IN_MODE>(tn, geom);
          if (lane == 0) mbar_arrive_expect_tx(&bars[sp], L::TILEB / P * nb);
          group_sync<NW>(grp);
          if (lane < P) my_offs[sp * P + lane] = pref;
          gather_io<T, H, W, P>(true, ring + sp * L::STAGEB, &in_map, &bars[sp], lane, nb, pref);
          const int64_t tq = tn + gstride;  // prefetch the next refill's offsets
          pref = (tq < ntiles && lane < tile_blocks<P, IN_MODE>(tq, geom))
                     ? geom.offsets[tq * P + lane] : 0;
        }
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

// Shared-ring producer / consumer kernel (LINEAR blocks, one block per stage):
// NC compute warps + 1 TMA producer warp per CTA, one CTA per SM, an S-stage ring
// SHARED by the compute warps (tile i of the CTA -> stage i % S, warp i % NC).
// The ring depth is decoupled from the warp count, which is what the 64x64 fp32
// tiles need: packed (FFMA2) 64-point passes hold two rows / two columns per
// lane (~200 registers), so only ~8 warps fit, and with the tile kernel's
// per-warp rings each of them would need >= 2 private 16 KB stages.
//   producer (lane 0): loads S tiles ahead; for each tile in order waits done[s],
//     issues the TMA store, and refills the previous tile's stage once its store
//     has been read (cp.async.bulk.wait_group.read 1)
//   compute warp: waits full[s], row + column pass in place (packed pairs),
//     fence.proxy.async, arrives done[s]
#ifndef DCTADJ_RING_PAIR
#define DCTADJ_RING_PAIR 1
#endif

template <typename T, int H, int W, int RC, int CC, bool COL_FIRST, int NC, int S>
__global__ void __launch_bounds__((NC + 1) * 32, 1)
    ring_kernel(const __grid_constant__ CUtensorMap in_map,
                const __grid_constant__ CUtensorMap out_map, const __grid_constant__ Geom geom,
                const __grid_constant__ KParams<T, W, H, RC, CC> prm) {
  using L = TileLayout<T, H, W, 1>;
  using RowOp = AxisOp<T, W, RC>;
  using ColOp = AxisOp<T, H, CC>;
  static_assert(!RowOp::kDense && !ColOp::kDense, "dense ops use the tile kernel");
  static_assert(sizeof(T) == 4 && L::PH == 64 && W == 64, "packed pairs over 64 rows / columns");
  static_assert(S >= NC, "the stage hand-off below relies on S >= NC");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::STAGEB);
  uint64_t* done = full + S;
  if (!geom.early) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], 1);
    }
    fence_mbar_init();
    prefetch_map(&in_map);
    prefetch_map(&out_map);
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  const int64_t n = geom.ntiles > blockIdx.x ? (geom.ntiles - blockIdx.x + G - 1) / G : 0;
  constexpr int GSQ = RowOp::kGainSq * ColOp::kGainSq;
  if (warp == NC) {
    if (lane == 0) {
      auto load = [&](int64_t i) {
        const int s = static_cast<int>(i % S);
        mbar_arrive_expect_tx(&full[s], L::TILEB);
        issue_tile_io<T, H, W, 1, MODE_LINEAR>(true, smem + s * L::STAGEB, &in_map, &full[s],
                                               blockIdx.x + i * G, geom, 1);
      };
      for (int64_t i = 0; i < S && i < n; ++i) load(i);
      for (int64_t i = 0; i < n; ++i) {
        const int s = static_cast<int>(i % S);
        mbar_wait(&done[s], static_cast<uint32_t>((i / S) & 1));
        issue_tile_io<T, H, W, 1, MODE_LINEAR>(false, smem + s * L::STAGEB, &out_map, nullptr,
                                               blockIdx.x + i * G, geom, 1);
        bulk_commit();
        if (i >= 1 && i - 1 + S < n) {  // tile i-1's stage: its store has been read
          bulk_wait_read<1>();
          load(i - 1 + S);
        }
      }
      bulk_wait_all();
    }
    if (geom.early) asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  for (int64_t i = warp; i < n; i += NC) {
    const int s = static_cast<int>(i % S);
    const int64_t k = i / S;  // this is the k-th use of stage s
    uint8_t* buf = smem + s * L::STAGEB;
    // A parity wait cannot tell phase k-1 from phase k+1.  Stage s's previous tile
    // (i - S) belongs to ANOTHER warp, so nothing this warp did orders it before
    // tile i: if its TMA load completed after the later-issued load of this warp's
    // previous tile (i - NC), full[s] would still be at phase k-1 here and the
    // parity-k wait would pass on the stale phase.  Waiting first for done[s] of
    // tile i - S (phase k-1) closes that: tile i - 2S is always consumed by now
    // (the producer issued load(i - NC) after done(i - NC - S + 1), and
    // i - NC - S + 1 > i - 2S since S >= NC), so done[s] is at phase k-1 or later
    // and this wait is exact; after it, full[s] is at phase k or k+1, and so is
    // the wait below.
    if (k >= 1) mbar_wait(&done[s], static_cast<uint32_t>((k - 1) & 1));
    mbar_wait(&full[s], static_cast<uint32_t>(k & 1));
    // Column-first (inverse) kernels: the two compute warps of an SM sub-partition (warps w
    // and w + 4) start their tiles together, so they walk the straight-line pass code
    // roughly in step and share its instruction fetches (the 64-point passes are ~75 KB of
    // code and instruction fetch is this kernel's top stall): inverse -1.5..-3 %; the
    // row-first kernels lose 14 % to it (both warps in their load / store phases at once)
    // and run unpaired (profiles/r02_tuning.md).  Both warps have a tile in this round
    // iff tile r * 8 + w + 4 exists.
    if constexpr (COL_FIRST && NC == 8 && DCTADJ_RING_PAIR != 0) {
      if (warp >= 4 || i + 4 < n) asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp & 3)) : "memory");
    }
    if constexpr (!COL_FIRST) {
      row_pass<T, H, W, 1, RC, 1, true>(buf, lane, prm.row, nullptr);
      __syncwarp();
      col_pass<T, H, W, 1, CC, GSQ, true>(buf, lane, prm.col, nullptr);
    } else {
      col_pass<T, H, W, 1, CC, 1, true>(buf, lane, prm.col, nullptr);
      __syncwarp();
      row_pass<T, H, W, 1, RC, GSQ, true>(buf, lane, prm.row, nullptr);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&done[s]);
  }
  if (geom.early) asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace dctadj

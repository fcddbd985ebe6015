// frames_exact.cuh -- config 5's comparison step in one kernel, warp-specialised
// with per-role register budgets (setmaxnreg).
//
// One HBM read of each frame super-tile (4 horizontally adjacent 32x32 blocks,
// one 4-D TMA box, row-interleaved in shared memory) feeds
//   * the EXACT transform Y_e = Dv X Dh^T on the tensor cores (3xTF32 tcgen05,
//     the dense_tc.cuh pipeline: A operand in TMEM, Dv / Dh hi / lo in smem),
//   * the ADJUSTED transform (row op FRC, column op FCC: the tile kernel's
//     register butterflies, packed FFMA2 row pairs and column pairs), and
//   * the per-frame approximation error sums of Y_a against Y_e.
//
// Warp roles (20 warps, one CTA per SM, 640 threads -> 96 registers at launch):
//   warps  0..7   2 exact-epilogue groups of 4 warps (96 registers), each with
//                 two tiles in flight (TMEM slots; B(i) / A(i+1) / C(i)): TMEM A
//                 operands, the W transpose, Y_e out of TMEM, the error sums,
//                 the TMA store of Y_e
//   warps  8..15  the adjusted warps, two warpgroups (setmaxnreg.inc -> 128
//                 registers, the budget of the packed 32-point passes): pair m
//                 takes tiles k = m (mod 4), each warp of the pair one half (2
//                 blocks) -- packed row pass from the ring stage into its own
//                 8 KB tile, packed column pass in place, TMA store of Y_a
//   warp  16      TMA producer (ring of S stages, dynamic chunked tile counter)
//   warps 17, 18  MMA issuers for pass 1 / pass 2 (blocking mbarrier waits)
//   warp  19      idle (completes the control warpgroup for setmaxnreg.dec -> 24)
//
// MEASURED SLOWER than the single-role fused kernel (dense_tc.cuh FUSED, the
// default; profiles/r02_c5_fused.md): 1.51-1.54 ms vs 1.45-1.48 ms for config 5.
// Built only with DCTADJ_TUNING=1 and selected by DCTADJ_FX_WS=1.  The exact
// side alone (adjusted math skipped) already takes 1.16-1.19 ms here -- the
// 2-group x 2-slot pipeline and the Y_a hand-off (adj_free) keep it latency-
// bound -- and the packed passes add ~0.35 ms on top.
//
// Hand-offs (mbarriers): full[s] (TMA), empty[s] (3 arrivals: the exact group
// after reading X for its A operand, each adjusted half after its row pass read
// X), a1_ready / d1_done / a2_ready / d2_done per exact group and TMEM slot,
// adj_done[m] (2 arrivals: Y_a of pair m's current tile complete) and
// adj_free[m] (the exact group has read Y_a; pair m may overwrite its tiles).
#pragma once
#include "dense_tc.cuh"

namespace dctadj {

constexpr int kFxGroups = 2;                  // exact-epilogue groups
constexpr int kFxAdjWarps = 8;                // adjusted warps: 4 pairs, one half-tile each
constexpr int kFxAdjSlots = kFxAdjWarps / 2;  // adjusted pairs (tile k -> pair k mod 4)

constexpr int kFxThreads = (4 * kFxGroups + kFxAdjWarps + 4) * 32;
constexpr int kFxAdjRegs = 128, kFxCtlRegs = 24;

DA_DEV void setmaxnreg_inc_adj() { asm volatile("setmaxnreg.inc.sync.aligned.u32 128;" ::: "memory"); }
DA_DEV void setmaxnreg_dec24() { asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory"); }

template <int S>
constexpr size_t frames_exact_smem() {
  return 1024 + static_cast<size_t>(S) * 16384 + 2 * kFxGroups * 16384 + kFxAdjWarps * 8192 + 16384 +
         (2 * S + 8 * kFxGroups + 2 * kFxAdjSlots) * 8 + (S + kFxGroups) * 8 + kFxGroups * 16 * 8 + 16;
}

template <int S, int FRC, int FCC>
__global__ void __launch_bounds__(kFxThreads, 1)
    frames_exact_kernel(const __grid_constant__ CUtensorMap in_map,
                        const __grid_constant__ CUtensorMap out_map,
                        const __grid_constant__ Geom geom, const __grid_constant__ DenseTcParams prm,
                        const __grid_constant__ CUtensorMap adj_map,
                        const __grid_constant__ KParams<float, 32, 32, FRC, FCC> kp) {
  constexpr int NG = kFxGroups, NA = kFxAdjWarps, NT = kFxAdjSlots;
  using RowOp = AxisOp<float, 32, FRC>;
  using ColOp = AxisOp<float, 32, FCC>;
  static_assert(!RowOp::kDense && !ColOp::kDense && !RowOp::kIdentity && !ColOp::kIdentity,
                "the adjusted side is a fast path on both axes");
  static_assert(S > NT && NT >= NG, "end markers: one per exact group and adjusted pair, no wrap");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stages = smem;                    // S x 16 KB: X super-tiles as loaded
  uint8_t* gtile = stages + S * 16384;       // 2 NG x 16 KB: W transpose / Y_e staging
  uint8_t* atile = gtile + 2 * NG * 16384;       // NA x 8 KB: Y_a half-tiles (2 blocks each)
  uint8_t* bmat = atile + NA * 8192;         // Dv hi/lo, Dh hi/lo
  uint8_t* dv_hi = bmat;
  uint8_t* dv_lo = bmat + 4096;
  uint8_t* dh_hi = bmat + 8192;
  uint8_t* dh_lo = bmat + 12288;
  uint64_t* full = reinterpret_cast<uint64_t*>(bmat + 16384);
  uint64_t* empty = full + S;
  uint64_t* a1_ready = empty + S;  // [2 g + slot]
  uint64_t* d1_done = a1_ready + 2 * NG;
  uint64_t* a2_ready = d1_done + 2 * NG;
  uint64_t* d2_done = a2_ready + 2 * NG;
  uint64_t* adj_done = d2_done + 2 * NG;
  uint64_t* adj_free = adj_done + NT;
  int64_t* tile_id = reinterpret_cast<int64_t*>(adj_free + NT);  // per stage; -1 = end
  // per exact group: the tile index of its end marker (set before its arrivals)
  volatile int64_t* mma_end = tile_id + S;
  double* red = reinterpret_cast<double*>(tile_id + S + NG);  // NG x 4 warps x 4
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red + NG * 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int e = tid; e < 1024; e += kFxThreads) {
    const int r = e >> 5, c = e & 31;
    const float h = prm.dh[e], v = prm.dv[e];
    const uint32_t hh = tc::tf32_hi(h), vh = tc::tf32_hi(v);
    *reinterpret_cast<uint32_t*>(dh_hi + tc::sw(r, c)) = hh;
    *reinterpret_cast<float*>(dh_lo + tc::sw(r, c)) = h - __uint_as_float(hh);
    *reinterpret_cast<uint32_t*>(dv_hi + tc::sw(r, c)) = vh;
    *reinterpret_cast<float*>(dv_lo + tc::sw(r, c)) = v - __uint_as_float(vh);
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 3);  // the exact group + both halves' adjusted warps
    }
    for (int g = 0; g < 2 * NG; ++g) {
      mbar_init(&a1_ready[g], 1);
      mbar_init(&d1_done[g], 1);
      mbar_init(&a2_ready[g], 1);
      mbar_init(&d2_done[g], 1);
    }
    for (int a = 0; a < NT; ++a) {
      mbar_init(&adj_done[a], 2);
      mbar_init(&adj_free[a], 1);
    }
    for (int g = 0; g < NG; ++g) mma_end[g] = INT64_MAX;
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the above overlaps the previous kernel
  const int64_t ntiles = geom.ntiles;
  constexpr int GSQ = RowOp::kGainSq * ColOp::kGainSq;

  if (warp >= 4 * NG + NA) {
    setmaxnreg_dec24();
    if (warp == 4 * NG + NA && lane == 0) {
      // ---------------- TMA producer: chunks of CH tiles (blockIdx.x, then a
      // global counter; the next chunk's atomic in flight while this one loads)
      constexpr int CH = 4;
      int64_t k = 0;
      int64_t chunk = blockIdx.x;
      unsigned long long nxt = atomicAdd(prm.sched, 1ull);
      for (;;) {
        const int64_t t0 = chunk * CH;
        if (t0 >= ntiles) break;
        for (int64_t t = t0; t < t0 + CH && t < ntiles; ++t, ++k) {
          const int s = static_cast<int>(k % S);
          mbar_wait(&empty[s], static_cast<uint32_t>(((k / S) & 1) ^ 1));
          tile_id[s] = t;
          mbar_arrive_expect_tx(&full[s], 16384);
          tc_tile_io<MODE_FRAME4>(true, stages + s * 16384, &in_map, &full[s], t, geom);
        }
        chunk = gridDim.x + static_cast<int64_t>(nxt);
        if (chunk * CH < ntiles) nxt = atomicAdd(prm.sched, 1ull);
      }
      asm volatile("griddepcontrol.launch_dependents;" :::);
      // end markers for tile indices k .. k + NT - 1: every exact group (k mod NG)
      // and every adjusted pair (k mod NT) meets one at its next tile
      for (int j = 0; j < NT; ++j, ++k) {
        const int s = static_cast<int>(k % S);
        mbar_wait(&empty[s], static_cast<uint32_t>(((k / S) & 1) ^ 1));
        tile_id[s] = -1;
        mbar_arrive(&full[s]);
      }
    } else if ((warp == 4 * NG + NA + 1 || warp == 4 * NG + NA + 2) && lane == 0) {
      // ---------------- MMA issuers: pass 1 / pass 2, each in tile order
      const bool pass1 = warp == 4 * NG + NA + 1;
      uint64_t* ready = pass1 ? a1_ready : a2_ready;
      uint64_t* done = pass1 ? d1_done : d2_done;
      const uint8_t* bhi = pass1 ? dv_hi : dh_hi;
      const uint8_t* blo = pass1 ? dv_lo : dh_lo;
      const uint32_t dcol = pass1 ? 64 : 96;
      // blocking waits (no polling beside the adjusted warps): an exact group that
      // meets its end marker sets mma_end[g] and arrives on both ready barriers
      for (int64_t k = 0;; ++k) {
        const int g = static_cast<int>(k % NG);
        const int64_t i = k / NG;
        const int u = static_cast<int>(i & 1);
        mbar_wait(&ready[2 * g + u], static_cast<uint32_t>((i >> 1) & 1));
        if (k >= mma_end[g]) break;  // group g's end marker (set before its arrivals)
        tc::fence_after();
        const uint32_t base = tmem + 256 * g + 128 * u;
        tc::gemm3_ts(base + dcol, base, bhi, blo);
        tc::commit(&done[2 * g + u]);
      }
    }
  } else if (warp >= 4 * NG) {
    // ---------------- adjusted warps: packed register butterflies on half-tiles.
    // Pair m = a / 2 takes tiles k = m (mod NT); half h = a % 2 transforms blocks
    // 2h, 2h + 1 of the super-tile (stage rows 4 r + 2 h + b') into its own 8 KB
    // block-major tile (row 32 b' + r); packed column pass from that tile into
    // registers, Y_a stored to HBM straight from registers.  No hand-off back
    // from the exact side: the ring alone paces the pairs.  Lane ->
    // (r, b') is chosen so that the 8 lanes of a 16-byte phase store 8 distinct
    // rows mod 8 (conflict-free) and load 4 distinct stage rows mod 8 (the most a
    // half super-tile offers: 2-way).
    setmaxnreg_inc_adj();
    const int a = warp - 4 * NG, m = a >> 1, h = a & 1;
    uint8_t* yt = atile + a * 8192;
    using L2 = TileLayout<float, 32, 32, 2>;
    for (int64_t j = 0;; ++j) {
      const int64_t k = m + NT * j;
      const int s = static_cast<int>(k % S);
      // the stage's previous tile belongs to other consumers: wait for its release
      // before the parity wait on full[s] (ring_kernel in tile_kernel.cuh)
      if (k >= S) mbar_wait(&empty[s], static_cast<uint32_t>(((k / S) - 1) & 1));
      mbar_wait(&full[s], static_cast<uint32_t>((k / S) & 1));
      const int64_t t = tile_id[s];
      if (t < 0) break;
      if (j > 0) {  // Y_a of this pair's previous tile read (error sums) and stored
        mbar_wait(&adj_free[m], static_cast<uint32_t>((j - 1) & 1));
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
      // an opaque copy of the lane index per tile: the swizzled addresses are
      // recomputed (a few integer ops) instead of being hoisted and spilled
      uint32_t ln;
      asm volatile("mov.u32 %0, %1;" : "=r"(ln) : "r"(lane));
      {  // row pass, block rows r0 and r0 + 16 packed (f2 lanes)
        const uint8_t* x = stages + s * 16384;
        f2 v[32];
        const uint32_t bb = ((ln >> 3) ^ (ln >> 1)) & 1;
        const uint32_t r0 = (ln & 7) | ((ln >> 4) << 3), r1 = r0 + 16;
        const uint32_t i0 = 4 * r0 + 2 * h + bb, i1 = 4 * r1 + 2 * h + bb;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 p0 = *reinterpret_cast<const float4*>(x + L2::addr(i0, q * 16));
          const float4 p1 = *reinterpret_cast<const float4*>(x + L2::addr(i1, q * 16));
          v[4 * q + 0].v = make_float2(p0.x, p1.x);
          v[4 * q + 1].v = make_float2(p0.y, p1.y);
          v[4 * q + 2].v = make_float2(p0.z, p1.z);
          v[4 * q + 3].v = make_float2(p0.w, p1.w);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // done with X
        apply_axis<f2, 32, FRC>(v, kp.row, nullptr);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          *reinterpret_cast<float4*>(yt + L2::addr(32 * bb + r0, q * 16)) =
              make_float4(v[4 * q].v.x, v[4 * q + 1].v.x, v[4 * q + 2].v.x, v[4 * q + 3].v.x);
          *reinterpret_cast<float4*>(yt + L2::addr(32 * bb + r1, q * 16)) =
              make_float4(v[4 * q].v.y, v[4 * q + 1].v.y, v[4 * q + 2].v.y, v[4 * q + 3].v.y);
        }
      }
      __syncwarp();
      col_pass<float, 32, 32, 2, FCC, GSQ, true, 32, false>(yt, ln, kp.col, nullptr);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&adj_map, yt, 0, static_cast<int>((4 * t + 2 * h) * 32));
        bulk_commit();
        mbar_arrive(&adj_done[m]);
      }
    }
    if (lane == 0) bulk_wait_all();
  } else {
    // ---------------- exact-epilogue groups, two tiles in flight per group.
    // Tile i of group g (k = g + NG i) uses slot u = i % 2: TMEM columns
    // 256 g + 128 u (A hi / lo +0..63, D1 +64, D2 +96) and staging tile gt[u].
    // Per iteration: B(i) (pass-1 result -> transpose -> pass-2 A), A(i+1) (the
    // next tile's pass-1 A), C(i) (Y_e, error sums, store): the MMA round trips
    // of one tile hide behind the other tile's work.
    const int g = warp >> 2;
    const uint32_t b = warp & 3;  // block of the super-tile = TMEM lane quadrant
    const uint32_t lane_addr = (b * 32) << 16;
    const bool leader = b == 0 && lane == 0;
    auto group_bar = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory"); };
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int acc_f = -1;
    auto flush = [&]() {
      if (acc_f >= 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double v = acc[i];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) red[(g * 4 + b) * 4 + i] = v;
        }
        group_bar();
        if (b == 0 && lane < 4)
          atomicAdd(prm.err + 4 * acc_f + lane, red[(g * 4 + 0) * 4 + lane] + red[(g * 4 + 1) * 4 + lane] +
                                                    red[(g * 4 + 2) * 4 + lane] + red[(g * 4 + 3) * 4 + lane]);
        group_bar();
      }
      acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
    };
    uint32_t v[32];
    // A(i): the tile's X column -> pass-1 A operand; returns its tile id (-1: end)
    auto stage_a = [&](int64_t i) -> int64_t {
      const int64_t k = g + NG * i;
      const int u = static_cast<int>(i & 1);
      const int s = static_cast<int>(k % S);
      if (k >= S) mbar_wait(&empty[s], static_cast<uint32_t>(((k / S) - 1) & 1));  // as above
      mbar_wait(&full[s], static_cast<uint32_t>((k / S) & 1));
      const int64_t t = tile_id[s];
      if (t < 0) {  // release the MMA issuers waiting for this tile index
        if (leader) {
          mma_end[g] = k;
          mbar_arrive(&a1_ready[2 * g + u]);
          mbar_arrive(&a2_ready[2 * g + u]);
        }
        return -1;
      }
      const uint8_t* x = stages + s * 16384;
      // pass-1 A: column j = lane of block b, A[(b,j)][i] = X_b[i][j]
#pragma unroll
      for (int r = 0; r < 32; ++r)
        v[r] = *reinterpret_cast<const uint32_t*>(x + tc::sw(tc_row<MODE_FRAME4>(b, r), lane));
      tc::st_split(tmem + 256 * g + 128 * u + lane_addr, v);
      tc::wait_st();
      tc::fence_before();
      group_bar();
      if (leader) {
        mbar_arrive(&empty[s]);  // done with X
        mbar_arrive(&a1_ready[2 * g + u]);
      }
      return t;
    };
    int64_t t = stage_a(0);
    for (int64_t i = 0; t >= 0; ++i) {
      const int u = static_cast<int>(i & 1);
      const uint32_t par = static_cast<uint32_t>((i >> 1) & 1);
      const uint32_t ta = tmem + 256 * g + 128 * u + lane_addr;
      uint8_t* gt = gtile + (2 * g + u) * 16384;
      // B(i): W_b = Dv X_b, lane j holds column j; transpose through this warp's 4 KB
      // (gt[u] is free: C(i-1) waited for the store of C(i-2))
      mbar_wait(&d1_done[2 * g + u], par);
      tc::fence_after();
      tc::ld32(ta + 64, v);
#pragma unroll
      for (int r = 0; r < 32; ++r) *reinterpret_cast<uint32_t*>(gt + tc::sw(b * 32 + r, lane)) = v[r];
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 w = *reinterpret_cast<const uint4*>(gt + tc::sw(b * 32 + lane, q * 4));
        v[4 * q] = w.x;
        v[4 * q + 1] = w.y;
        v[4 * q + 2] = w.z;
        v[4 * q + 3] = w.w;
      }
      tc::st_split(ta, v);  // pass-2 A: row r = lane, A[(b,r)][j] = W_b[r][j]
      tc::wait_st();
      tc::fence_before();
      group_bar();
      if (leader) mbar_arrive(&a2_ready[2 * g + u]);
      // A(i+1) while pass 2 of tile i runs
      const int64_t t_next = stage_a(i + 1);
      // C(i): Y_e rows out of TMEM; error of this row against Y_a (the adjusted pair)
      const int64_t k = g + NG * i;
      mbar_wait(&d2_done[2 * g + u], par);
      tc::fence_after();
      tc::ld32(ta + 96, v);
      const int aw = static_cast<int>(k % NT);
      // block b of the tile: half b / 2 of pair aw, row 32 (b % 2) + lane
      const uint8_t* ya_t = atile + (2 * aw + (b >> 1)) * 8192;
      mbar_wait(&adj_done[aw], static_cast<uint32_t>((k / NT) & 1));
      float d2 = 0.f, e2 = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 ya4 = *reinterpret_cast<const float4*>(ya_t + tc::sw((b & 1) * 32 + lane, q * 4));
        const float ya[4] = {ya4.x, ya4.y, ya4.z, ya4.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float ye = __uint_as_float(v[4 * q + w]), d = ya[w] - ye;
          d2 = fmaf(d, d, d2);
          e2 = fmaf(ye, ye, e2);
        }
      }
      const int64_t per = static_cast<int64_t>(geom.tiles_x) * geom.tiles_y, blk = 4 * t;
      const int f = static_cast<int>(blk / per);
      const int ty = static_cast<int>((blk - f * per) / geom.tiles_x);
      if (f != acc_f) {
        flush();
        acc_f = f;
      }
      acc[0] += d2;
      acc[1] += e2;
      if ((ty + 1) * 32 <= prm.frame_h) {
        acc[2] += d2;
        acc[3] += e2;
      }
      // Y_e staged in gt[u] (row (b, lane)), one TMA store per tile
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint4*>(gt + tc::sw(tc_row<MODE_LINEAR>(b, lane), q * 4)) =
            make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      fence_proxy_async_smem();
      if (leader) bulk_wait_read<0>();  // Y_e(i-1) has left gt[1-u] (B(i+1) writes it next)
      group_bar();
      if (leader) {
        mbar_arrive(&adj_free[aw]);  // the whole group has read Y_a
        tc_tile_io<MODE_LINEAR>(false, gt, &out_map, nullptr, t, geom);
        bulk_commit();
      }
      t = t_next;
    }
    flush();
    if (leader) bulk_wait_all();
  }
  tc::fence_before();
  __syncthreads();
  if (tid == 0) {  // the last CTA out re-arms the tile counter for the next launch
    __threadfence();
    if (atomicAdd(prm.sched + 1, 1ull) == gridDim.x - 1) {
      prm.sched[0] = 0;
      prm.sched[1] = 0;
      __threadfence();
    }
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace dctadj

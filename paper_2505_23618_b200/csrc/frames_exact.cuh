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
//   warps  0..11  3 exact-epilogue groups of 4 warps (96 registers): TMEM A
//                 operands, the W transpose, Y_e out of TMEM, the error sums,
//                 the TMA store of Y_e; group g takes tiles k = g (mod 3)
//   warps 12..15  the adjusted warpgroup (setmaxnreg.inc -> 168 registers, the
//                 budget the packed 32-point passes need): warp a takes tiles
//                 k = a (mod 4) whole -- row pass from the ring stage into its own
//                 16 KB tile, column pass in place, TMA store of Y_a
//   warp  16      TMA producer (ring of S stages, dynamic chunked tile counter)
//   warps 17, 18  MMA issuers for pass 1 / pass 2
//   warp  19      idle (completes the control warpgroup for setmaxnreg.dec -> 24)
// The earlier single-role fused kernel ran the adjusted butterflies in the
// exact epilogue's warps at 96 registers, i.e. in scalar lanes, and was issue-
// bound (0.64 of the HBM roofline); splitting the roles lets the adjusted
// passes run packed while the exact epilogue keeps its latency hiding.
//
// Hand-offs (mbarriers): full[s] (TMA), empty[s] (2 arrivals: the exact group
// after reading X for its A operand, the adjusted warp after its row pass read
// X), a1_ready / d1_done / a2_ready / d2_done per exact group, adj_done[a]
// (Y_a of warp a's current tile complete in its tile) and adj_free[a] (the exact
// group has read Y_a for the error sums; warp a may overwrite its tile).
#pragma once
#include "dense_tc.cuh"

namespace dctadj {

constexpr int kFxGroups = 3;                  // exact-epilogue groups
constexpr int kFxAdjWarps = 4;                // adjusted warpgroup
constexpr int kFxThreads = (4 * kFxGroups + kFxAdjWarps + 4) * 32;
constexpr int kFxAdjRegs = 168, kFxCtlRegs = 24;

DA_DEV void setmaxnreg_inc168() { asm volatile("setmaxnreg.inc.sync.aligned.u32 168;" ::: "memory"); }
DA_DEV void setmaxnreg_dec24() { asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory"); }

template <int S>
constexpr size_t frames_exact_smem() {
  return 1024 + static_cast<size_t>(S) * 16384 + kFxGroups * 16384 + kFxAdjWarps * 16384 + 16384 +
         (2 * S + 4 * kFxGroups + 2 * kFxAdjWarps) * 8 + (S + 1) * 8 + kFxGroups * 16 * 8 + 16;
}

template <int S, int FRC, int FCC>
__global__ void __launch_bounds__(kFxThreads, 1)
    frames_exact_kernel(const __grid_constant__ CUtensorMap in_map,
                        const __grid_constant__ CUtensorMap out_map,
                        const __grid_constant__ Geom geom, const __grid_constant__ DenseTcParams prm,
                        const __grid_constant__ CUtensorMap adj_map,
                        const __grid_constant__ KParams<float, 32, 32, FRC, FCC> kp) {
  constexpr int NG = kFxGroups, NA = kFxAdjWarps;
  using RowOp = AxisOp<float, 32, FRC>;
  using ColOp = AxisOp<float, 32, FCC>;
  static_assert(!RowOp::kDense && !ColOp::kDense && !RowOp::kIdentity && !ColOp::kIdentity,
                "the adjusted side is a fast path on both axes");
  static_assert(S > NA, "end markers must not wrap the ring");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stages = smem;                    // S x 16 KB: X super-tiles as loaded
  uint8_t* gtile = stages + S * 16384;       // NG x 16 KB: W transpose / Y_e staging
  uint8_t* atile = gtile + NG * 16384;       // NA x 16 KB: Y_a per adjusted warp
  uint8_t* bmat = atile + NA * 16384;        // Dv hi/lo, Dh hi/lo
  uint8_t* dv_hi = bmat;
  uint8_t* dv_lo = bmat + 4096;
  uint8_t* dh_hi = bmat + 8192;
  uint8_t* dh_lo = bmat + 12288;
  uint64_t* full = reinterpret_cast<uint64_t*>(bmat + 16384);
  uint64_t* empty = full + S;
  uint64_t* a1_ready = empty + S;
  uint64_t* d1_done = a1_ready + NG;
  uint64_t* a2_ready = d1_done + NG;
  uint64_t* d2_done = a2_ready + NG;
  uint64_t* adj_done = d2_done + NG;
  uint64_t* adj_free = adj_done + NA;
  int64_t* tile_id = reinterpret_cast<int64_t*>(adj_free + NA);  // per stage; -1 = end
  volatile int64_t* total_k = tile_id + S;
  double* red = reinterpret_cast<double*>(tile_id + S + 1);  // NG x 4 warps x 4
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
      mbar_init(&empty[s], 2);
    }
    for (int g = 0; g < NG; ++g) {
      mbar_init(&a1_ready[g], 1);
      mbar_init(&d1_done[g], 1);
      mbar_init(&a2_ready[g], 1);
      mbar_init(&d2_done[g], 1);
    }
    for (int a = 0; a < NA; ++a) {
      mbar_init(&adj_done[a], 1);
      mbar_init(&adj_free[a], 1);
    }
    *total_k = -1;
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
      *total_k = k;
      asm volatile("griddepcontrol.launch_dependents;" :::);
      // end markers for tile indices k .. k + NA - 1: every exact group (k mod NG)
      // and every adjusted warp (k mod NA) meets one at its next tile
      for (int j = 0; j < NA; ++j, ++k) {
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
      for (int64_t k = 0;; ++k) {
        const int g = static_cast<int>(k % NG);
        const uint32_t par = static_cast<uint32_t>((k / NG) & 1);
        bool ok;
        while (!(ok = mbar_test(&ready[g], par))) {
          const int64_t tot = *total_k;
          if (tot >= 0 && k >= tot) break;
        }
        if (!ok) break;
        tc::fence_after();
        tc::gemm3_ts(tmem + 128 * g + dcol, tmem + 128 * g, bhi, blo);
        tc::commit(&done[g]);
      }
    }
  } else if (warp >= 4 * NG) {
    // ---------------- adjusted warpgroup: packed register butterflies
    setmaxnreg_inc168();
    const int a = warp - 4 * NG;
    uint8_t* yt = atile + a * 16384;
    for (int64_t j = 0;; ++j) {
      const int64_t k = a + NA * j;
      const int s = static_cast<int>(k % S);
      mbar_wait(&full[s], static_cast<uint32_t>((k / S) & 1));
      const int64_t t = tile_id[s];
      if (t < 0) break;
      if (j > 0) {  // this warp's tile: Y_a of its previous tile read (error sums) and stored
        mbar_wait(&adj_free[a], static_cast<uint32_t>((j - 1) & 1));
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
      row_pass_io<float, 32, 32, 4, FRC, 1, true, 32>(stages + s * 16384, yt, lane, kp.row,
                                                       nullptr);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // done with X
      col_pass<float, 32, 32, 4, FCC, GSQ, true, 32, true>(yt, lane, kp.col, nullptr);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(&adj_map, yt, 0, static_cast<int>(4 * t), 0);
        bulk_commit();
        mbar_arrive(&adj_done[a]);
      }
    }
    if (lane == 0) bulk_wait_all();
  } else {
    // ---------------- exact-epilogue groups
    const int g = warp >> 2;
    const uint32_t b = warp & 3;  // block of the super-tile = TMEM lane quadrant
    const uint32_t lane_addr = (b * 32) << 16;
    const bool leader = b == 0 && lane == 0;
    uint8_t* gt = gtile + g * 16384;
    const uint32_t ta = tmem + 128 * g + lane_addr;
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
    for (int64_t k = g;; k += NG) {
      const int s = static_cast<int>(k % S);
      const uint32_t gp = static_cast<uint32_t>((k / NG) & 1);
      const uint8_t* x = stages + s * 16384;
      uint32_t v[32];
      mbar_wait(&full[s], static_cast<uint32_t>((k / S) & 1));
      const int64_t t = tile_id[s];
      if (t < 0) break;
      // pass-1 A: column j = lane of block b, A[(b,j)][i] = X_b[i][j]
#pragma unroll
      for (int i = 0; i < 32; ++i)
        v[i] = *reinterpret_cast<const uint32_t*>(x + tc::sw(tc_row<MODE_FRAME4>(b, i), lane));
      tc::st_split(ta, v);
      tc::wait_st();
      if (leader) bulk_wait_read<0>();  // Y_e(k - NG) has left the group tile
      tc::fence_before();
      group_bar();
      if (leader) {
        mbar_arrive(&empty[s]);  // done with X
        mbar_arrive(&a1_ready[g]);
      }
      // W_b = Dv X_b: lane j holds column j; transpose through this warp's 4 KB
      mbar_wait(&d1_done[g], gp);
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
      if (leader) mbar_arrive(&a2_ready[g]);
      // Y_e rows out of TMEM; error of this row against Y_a (the adjusted warp's tile)
      mbar_wait(&d2_done[g], gp);
      tc::fence_after();
      tc::ld32(ta + 96, v);
      const int aw = static_cast<int>(k % NA);
      const uint8_t* ya_t = atile + aw * 16384;
      mbar_wait(&adj_done[aw], static_cast<uint32_t>((k / NA) & 1));
      float d2 = 0.f, e2 = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 ya4 = *reinterpret_cast<const float4*>(ya_t + tc::sw(lane * 4 + b, q * 4));
        const float ya[4] = {ya4.x, ya4.y, ya4.z, ya4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float ye = __uint_as_float(v[4 * q + u]), d = ya[u] - ye;
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
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint4*>(gt + tc::sw(tc_row<MODE_LINEAR>(b, lane), q * 4)) =
            make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      fence_proxy_async_smem();
      tc::fence_before();
      group_bar();
      if (leader) {
        mbar_arrive(&adj_free[aw]);  // the whole group has read Y_a
        tc_tile_io<MODE_LINEAR>(false, gt, &out_map, nullptr, t, geom);
        bulk_commit();
      }
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

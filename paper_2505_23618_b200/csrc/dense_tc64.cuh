// dense_tc64.cuh -- the dense comparison path for 64x64 fp32 blocks on the
// tensor cores (same design as dense_tc.cuh's 32x32 kernel, scaled up):
//
//   pass 1  D1[(b,j)][r] = sum_i X_b[i][j] Dv[r][i]     M=128 (2 blocks x 64), N=64, K=64
//   pass 2  D2[(b,r)][n] = sum_j W_b[r][j] Dh[n][j]     W_b = Dv X_b;  Y_b[r][n] = D2[(b,r)][n]
//
// 3xTF32 (hi*hi + hi*lo + lo*hi), data operand A in TMEM (hi 64 + lo 64
// columns), the 64x64 coefficient matrices as smem B operands (hi/lo, 64 KB),
// super-tiles of 2 blocks (32 KB).  Two epilogue groups (TMEM: A 128 + D 64
// columns each, D1 and D2 sharing theirs), a TMA producer warp with a
// self-re-arming chunked tile counter, one MMA-issuer warp per pass.  The W
// transpose between the passes crosses the two warps of a block, so it goes
// through the group's 32 KB staging tile under the group barrier.
#pragma once
#include "dense_tc.cuh"

namespace dctadj {

constexpr int kTc64Groups = 2;
constexpr int kTc64Threads = (4 * kTc64Groups + 3) * 32;

namespace tc {
// instruction descriptor: D f32, A/B tf32, K-major, N = 64, M = 128
constexpr uint32_t kIdesc64 = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) |
                              ((128u >> 4) << 24);
DA_DEV void mma64_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(static_cast<uint32_t>(accumulate)), "r"(kIdesc64)
      : "memory");
}
// B: 64 (N) rows x 64 (K) tf32, K-major SW128 as two 8 KB K-slices (32 K each)
DA_DEV uint32_t sw64(uint32_t n, uint32_t k) { return (k >> 5) * 8192 + sw(n, k & 31); }
// D (+)= A_hi B_hi + A_hi B_lo + A_lo B_hi over K = 64
DA_DEV void gemm3_ts64(uint32_t tmem_d, uint32_t tmem_a, const uint8_t* bhi, const uint8_t* blo) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t off = (k >> 2) * 8192 + (k & 3) * 32;  // 8 tf32 = 32 bytes along K
    const uint64_t dbh = desc_k_sw128(bhi + off), dbl = desc_k_sw128(blo + off);
    mma64_ts(tmem_d, tmem_a + 8 * k, dbh, k > 0);
    mma64_ts(tmem_d, tmem_a + 8 * k, dbl, true);
    mma64_ts(tmem_d, tmem_a + 64 + 8 * k, dbh, true);
  }
}
// split 64 values into tf32 hi (columns taddr..+63) and lo (taddr+64..+127)
DA_DEV void st_split64(uint32_t taddr, uint32_t (&v)[64]) {
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint32_t hi[32], lo[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const float x = __uint_as_float(v[32 * half + c]);
      hi[c] = tf32_hi(x);
      lo[c] = __float_as_uint(x - __uint_as_float(hi[c]));
    }
    st32(taddr + 32 * half, hi);
    st32(taddr + 64 + 32 * half, lo);
  }
}
DA_DEV void ld64(uint32_t taddr, uint32_t (&v)[64]) {
  uint32_t a[32], b[32];
  ld32(taddr, a);
  ld32(taddr + 32, b);
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = a[c], v[32 + c] = b[c];
}
}  // namespace tc

template <int S>
__global__ void __launch_bounds__(kTc64Threads, 1)
    dense_tc64_kernel(const __grid_constant__ CUtensorMap in_map,
                      const __grid_constant__ CUtensorMap out_map, const __grid_constant__ Geom geom,
                      const __grid_constant__ DenseTcParams prm) {
  constexpr int NGRP = kTc64Groups;
  using L = TileLayout<float, 64, 64, 2>;  // 2 boxes (column slices) of 128 rows x 128 B
  static_assert(L::TILEB == 32768 && L::NB == 2, "2 blocks of 64x64 fp32");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stages = smem;                  // S x 32 KB: X tiles as loaded
  uint8_t* gtile = smem + S * 32768;       // NGRP x 32 KB: W transpose / Y staging
  uint8_t* bmat = gtile + NGRP * 32768;    // 4 x 16 KB: Dv hi/lo, Dh hi/lo
  uint8_t* dv_hi = bmat;
  uint8_t* dv_lo = bmat + 16384;
  uint8_t* dh_hi = bmat + 32768;
  uint8_t* dh_lo = bmat + 49152;
  uint64_t* full = reinterpret_cast<uint64_t*>(bmat + 65536);
  uint64_t* empty = full + S;
  uint64_t* a1_ready = empty + S;
  uint64_t* d1_done = a1_ready + NGRP;
  uint64_t* a2_ready = d1_done + NGRP;
  uint64_t* d2_done = a2_ready + NGRP;
  int64_t* tile_id = reinterpret_cast<int64_t*>(d2_done + NGRP);
  volatile int64_t* total_k = tile_id + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_id + S + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int e = tid; e < 4096; e += kTc64Threads) {
    const int r = e >> 6, c = e & 63;
    const float h = prm.dh[e], v = prm.dv[e];
    const uint32_t hh = tc::tf32_hi(h), vh = tc::tf32_hi(v);
    *reinterpret_cast<uint32_t*>(dh_hi + tc::sw64(r, c)) = hh;
    *reinterpret_cast<float*>(dh_lo + tc::sw64(r, c)) = h - __uint_as_float(hh);
    *reinterpret_cast<uint32_t*>(dv_hi + tc::sw64(r, c)) = vh;
    *reinterpret_cast<float*>(dv_lo + tc::sw64(r, c)) = v - __uint_as_float(vh);
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int g = 0; g < NGRP; ++g) {
      mbar_init(&a1_ready[g], 1);
      mbar_init(&d1_done[g], 1);
      mbar_init(&a2_ready[g], 1);
      mbar_init(&d2_done[g], 1);
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
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t ntiles = geom.ntiles;

  if (warp == 4 * NGRP) {
    // ---------------- TMA producer (chunks of 4 super-tiles from a global counter)
    if (lane == 0) {
      constexpr int CH = 4;
      int64_t k = 0, chunk = blockIdx.x;
      unsigned long long nxt = atomicAdd(prm.sched, 1ull);
      for (;;) {
        const int64_t t0 = chunk * CH;
        if (t0 >= ntiles) break;
        for (int64_t t = t0; t < t0 + CH && t < ntiles; ++t, ++k) {
          const int s = static_cast<int>(k % S);
          mbar_wait(&empty[s], static_cast<uint32_t>(((k / S) & 1) ^ 1));
          tile_id[s] = t;
          const int nb = tile_blocks<2, MODE_LINEAR>(t, geom);
          mbar_arrive_expect_tx(&full[s], 16384 * nb);
          issue_tile_io<float, 64, 64, 2, MODE_LINEAR>(true, stages + s * 32768, &in_map,
                                                       &full[s], t, geom, nb);
        }
        chunk = gridDim.x + static_cast<int64_t>(nxt);
        if (chunk * CH < ntiles) nxt = atomicAdd(prm.sched, 1ull);
      }
      *total_k = k;
      asm volatile("griddepcontrol.launch_dependents;" :::);
      for (int j = 0; j < NGRP; ++j, ++k) {
        const int s = static_cast<int>(k % S);
        mbar_wait(&empty[s], static_cast<uint32_t>(((k / S) & 1) ^ 1));
        tile_id[s] = -1;
        mbar_arrive(&full[s]);
      }
    }
  } else if (warp == 4 * NGRP + 1 || warp == 4 * NGRP + 2) {
    // ---------------- MMA issuers: pass 1 / pass 2, each in tile order
    const bool pass1 = warp == 4 * NGRP + 1;
    uint64_t* ready = pass1 ? a1_ready : a2_ready;
    uint64_t* done = pass1 ? d1_done : d2_done;
    const uint8_t* bhi = pass1 ? dv_hi : dh_hi;
    const uint8_t* blo = pass1 ? dv_lo : dh_lo;
    if (lane == 0) {
      for (int64_t k = 0;; ++k) {
        const int g = static_cast<int>(k % NGRP);
        const uint32_t par = static_cast<uint32_t>((k / NGRP) & 1);
        bool ok;
        while (!(ok = mbar_test(&ready[g], par))) {
          const int64_t tot = *total_k;
          if (tot >= 0 && k >= tot) break;
        }
        if (!ok) break;
        tc::fence_after();
        tc::gemm3_ts64(tmem + 256 * g + 128, tmem + 256 * g, bhi, blo);
        tc::commit(&done[g]);
      }
    }
  } else {
    // ---------------- epilogue groups: lane m = 32 (warp % 4) + lane = (block b, index j)
    const int g = warp >> 2;
    const uint32_t q = warp & 3, m = q * 32 + lane, b = m >> 6, j = m & 63;
    const uint32_t ta = tmem + 256 * g + ((q * 32) << 16);  // this lane's A; D at +128
    const bool leader = q == 0 && lane == 0;
    uint8_t* gt = gtile + g * 32768;
    auto group_bar = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory"); };
    for (int64_t k = g;; k += NGRP) {
      const int s = static_cast<int>(k % S);
      const uint32_t gp = static_cast<uint32_t>((k / NGRP) & 1);
      const uint8_t* x = stages + s * 32768;
      uint32_t v[64];
      // stage s's previous tile (k - S) belongs to the other group (S = 3, 2 groups):
      // wait for its release first, or a parity wait on full[s] could pass on the
      // stale phase if that older load completed after this group's previous one
      // (ring_kernel in tile_kernel.cuh has the full argument)
      if (k >= S) mbar_wait(&empty[s], static_cast<uint32_t>(((k / S) - 1) & 1));
      mbar_wait(&full[s], static_cast<uint32_t>((k / S) & 1));
      const int64_t t = tile_id[s];
      if (t < 0) break;
      // pass-1 A: A[(b,j)][i] = X_b[i][j]
#pragma unroll
      for (int i = 0; i < 64; ++i)
        v[i] = *reinterpret_cast<const uint32_t*>(x + L::addr(b * 64 + i, j * 4));
      tc::st_split64(ta, v);
      tc::wait_st();
      if (leader) bulk_wait_read<0>();  // Y(k - NGRP) has left the staging tile
      tc::fence_before();
      group_bar();
      if (leader) {
        mbar_arrive(&empty[s]);
        mbar_arrive(&a1_ready[g]);
      }
      // W_b = Dv X_b: lane (b, j) holds column j; transpose through the staging tile
      mbar_wait(&d1_done[g], gp);
      tc::fence_after();
      tc::ld64(ta + 128, v);
#pragma unroll
      for (int r = 0; r < 64; ++r) *reinterpret_cast<uint32_t*>(gt + L::addr(b * 64 + r, j * 4)) = v[r];
      group_bar();
#pragma unroll
      for (int c = 0; c < 64; c += 4) {
        const uint4 w = *reinterpret_cast<const uint4*>(gt + L::addr(b * 64 + j, c * 4));
        v[c] = w.x, v[c + 1] = w.y, v[c + 2] = w.z, v[c + 3] = w.w;
      }
      tc::st_split64(ta, v);  // pass-2 A: row r = j, A[(b,r)][c] = W_b[r][c]
      tc::wait_st();
      tc::fence_before();
      group_bar();
      if (leader) mbar_arrive(&a2_ready[g]);
      // Y_b rows from TMEM into the staging tile, TMA store
      mbar_wait(&d2_done[g], gp);
      tc::fence_after();
      tc::ld64(ta + 128, v);
#pragma unroll
      for (int c = 0; c < 64; c += 4)
        *reinterpret_cast<uint4*>(gt + L::addr(b * 64 + j, c * 4)) =
            make_uint4(v[c], v[c + 1], v[c + 2], v[c + 3]);
      fence_proxy_async_smem();
      tc::fence_before();
      group_bar();
      if (leader) {
        issue_tile_io<float, 64, 64, 2, MODE_LINEAR>(false, gt, &out_map, nullptr, t, geom,
                                                     tile_blocks<2, MODE_LINEAR>(t, geom));
        bulk_commit();
      }
    }
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

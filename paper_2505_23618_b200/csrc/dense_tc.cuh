// dense_tc.cuh -- the dense comparison path on the 5th-generation tensor cores.
//
// Y_b = Dv X_b Dh^T for 32x32 fp32 blocks (the exact DST-7 / DCT-8 of config 5,
// the naive five-transform encoder baseline, Table 1's full-matrix column), as
// two tcgen05.mma (kind::tf32) GEMMs per super-tile of 4 blocks, in 3xTF32
// (a = a_hi + a_lo; a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi: fp32-level error).
//
//   pass 1  D1[(b,j)][r] = sum_i X_b[i][j] Dv[r][i]     M=128 (4 blocks x 32), N=32, K=32
//   pass 2  D2[(b,r)][n] = sum_j W_b[r][j] Dh[n][j]     W_b = Dv X_b;  Y_b[r][n] = D2[(b,r)][n]
//
// The data operand (A) lives in TENSOR MEMORY, not shared memory: the kernel is
// bound by shared-memory bandwidth once HBM is streamed, and an smem A operand
// is re-read by every MMA of the 3xTF32 split.  Each epilogue thread owns one
// TMEM lane: it reads its column of the TMA-loaded block (conflict-free on the
// 128-byte swizzle), splits it into tf32 hi / lo and tcgen05.st's both into the
// A columns; after pass 1 it transposes W through a per-warp 4 KB smem tile and
// stores the pass-2 A operand the same way.  Only the 32x32 coefficient
// matrices (hi / lo, 16 KB) are smem (B) operands.  One elected thread issues
// the MMAs; completion is tcgen05.commit -> mbarrier.
#pragma once
#include "tile_kernel.cuh"

namespace dctadj {

namespace tc {

// tf32 "hi" part by truncation (low 13 mantissa bits cleared); x - hi is exact
// in fp32, and the tensor core reads both as tf32 (3xTF32 split)
DA_DEV uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

// K-major SW128 UMMA smem descriptor (start address >> 4, LBO 16 B, SBO 1024 B,
// version 1, layout SWIZZLE_128B); the tile base must be 1024-byte aligned.
DA_DEV uint64_t desc_k_sw128(const void* p) {
  const uint64_t a = (smem_u32(p) >> 4) & 0x3FFF;
  return a | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// instruction descriptor: D f32, A/B tf32, both K-major, N = 32, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) |
                            ((128u >> 4) << 24);

DA_DEV void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(static_cast<uint32_t>(accumulate)), "r"(kIdesc)
      : "memory");
}

DA_DEV void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
DA_DEV void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DA_DEV void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

DA_DEV void ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

DA_DEV void ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// byte offset of element (row, col) of a 128-row x 32-float SW128 tile
DA_DEV uint32_t sw(uint32_t row, uint32_t col) {
  const uint32_t a = row * 128 + col * 4;
  return a ^ (((a >> 7) & 7) << 4);
}

// D (+)= A_hi B_hi + A_hi B_lo + A_lo B_hi over K = 32 (4 k-steps of 8)
DA_DEV void gemm3(uint32_t tmem_d, const uint8_t* ahi, const uint8_t* alo, const uint8_t* bhi,
                  const uint8_t* blo) {
  const uint64_t dah = desc_k_sw128(ahi), dal = desc_k_sw128(alo);
  const uint64_t dbh = desc_k_sw128(bhi), dbl = desc_k_sw128(blo);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint64_t off = static_cast<uint64_t>(k * 32) >> 4;  // 8 tf32 = 32 bytes along K
    mma_tf32(tmem_d, dah + off, dbh + off, k > 0);
    mma_tf32(tmem_d, dah + off, dbl + off, true);
    mma_tf32(tmem_d, dal + off, dbh + off, true);
  }
}

}  // namespace tc

struct DenseTcParams {
  const float* dh;  // device 32x32: row-pass matrix (Y = Dv X Dh^T)
  const float* dv;  // device 32x32: column-pass matrix
  unsigned long long* trace;  // diagnostics (DCTADJ_TC_TRACE): CTA 0 event clocks, or null
  unsigned long long* sched;  // [next, done]: dynamic tile counter, zero between launches
  double* err;     // fused: per frame [sum d^2 all, sum e^2 all, sum d^2 full rows, sum e^2 full]
  int32_t frame_h; // fused: frame height (tile rows below it are zero-padded)
  int32_t spin_ns; // MMA issuers: back-off (ns, __nanosleep) between readiness polls; 0 = spin
};
constexpr int kTcTraceTiles = 128, kTcTraceEv = 8, kTcTraceCtas = 1024;
DA_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int kDenseTcGroups = 4;
constexpr int kDenseTcThreads = (4 * kDenseTcGroups + 3) * 32;

namespace tc {
// D (+)= A_hi B_hi + A_hi B_lo + A_lo B_hi over K = 32, A in TMEM (hi at
// columns a..a+31, lo at a+32..a+63; one tf32 per column, lane = row)
DA_DEV void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(static_cast<uint32_t>(accumulate)), "r"(kIdesc)
      : "memory");
}
DA_DEV void gemm3_ts(uint32_t tmem_d, uint32_t tmem_a, const uint8_t* bhi, const uint8_t* blo) {
  const uint64_t dbh = desc_k_sw128(bhi), dbl = desc_k_sw128(blo);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint64_t off = static_cast<uint64_t>(k * 32) >> 4;  // 8 tf32 = 32 bytes along K
    mma_tf32_ts(tmem_d, tmem_a + 8 * k, dbh + off, k > 0);
    mma_tf32_ts(tmem_d, tmem_a + 8 * k, dbl + off, true);
    mma_tf32_ts(tmem_d, tmem_a + 32 + 8 * k, dbh + off, true);
  }
}
DA_DEV void st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
DA_DEV void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// split v into tf32 hi / lo and store both into this thread's TMEM lane
DA_DEV void st_split(uint32_t taddr, uint32_t (&v)[32]) {
  uint32_t lo[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const uint32_t h = tf32_hi(__uint_as_float(v[c]));
    lo[c] = __float_as_uint(__uint_as_float(v[c]) - __uint_as_float(h));
    v[c] = h;
  }
  st32(taddr, v);
  st32(taddr + 32, lo);
}
}  // namespace tc

// super-tile t of the LINEAR / FRAME / FRAME4 side (4 blocks of 32 x 32 fp32)
template <int MODE>
DA_DEV void tc_tile_io(bool load, uint8_t* buf, const CUtensorMap* map, uint64_t* bar, int64_t t,
                       const Geom& g) {
  if constexpr (MODE == MODE_FRAME4) {
    const int64_t per = static_cast<int64_t>(g.tiles_x) * g.tiles_y, blk = 4 * t;
    const int f = static_cast<int>(blk / per);
    const int rem = static_cast<int>(blk - f * per);
    const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
    if (load)
      tma_load_4d(buf, map, bar, 0, tx, ty * 32, f);
    else
      tma_store_4d(map, buf, 0, tx, ty * 32, f);
  } else {
    issue_tile_io<float, 32, 32, 4, MODE>(load, buf, map, bar, t, g, tile_blocks<4, MODE>(t, g));
  }
}
// smem tile row of (block b, block row r)
template <int MODE>
DA_DEV uint32_t tc_row(uint32_t b, uint32_t r) {
  return MODE == MODE_FRAME4 ? r * 4 + b : b * 32 + r;
}

// Warp-specialised pipeline (one CTA per SM, 4 * NGRP + 3 warps):
//   warp 4*NGRP     TMA producer: S-stage ring of 4-block super-tiles (16 KB)
//   warps 4*NGRP+1, +2  MMA issuers (one lane each) for pass 1 / pass 2, in tile
//                   order, as soon as the owning group signals (two issuers: a
//                   single thread issuing 24 small MMAs per tile is the pace)
//   warps 0..4*NGRP-1  NGRP epilogue groups of 4 warps; group g handles tiles
//                   k = g (mod NGRP); warp w owns TMEM lane quadrant w % 4 (= block
//                   b of the super-tile), so a group covers all 128 lanes of its
//                   TMEM slot: A (hi, lo: 64 columns), D1 (32), D2 (32)
// Hand-offs are mbarriers: full/empty (ring), a1_ready / d1_done / a2_ready /
// d2_done per group; a group's threads meet at a named barrier before its
// elected thread arrives or issues the TMA store of Y (staged in the group's
// 16 KB smem tile, which also carries the per-warp W transposes).
//
// FUSED (FRC != 0; config 5): the same launch also runs the ADJUSTED transform
// (row op FRC, column op FCC, the tile kernel's register butterflies, scalar
// lanes, 128 threads per group) in place on the loaded frame super-tile while
// the MMAs are in flight, stores it through adj_map (block-major, interleaved
// tile), and accumulates the per-frame approximation error of adjusted vs exact
// coefficients -- one HBM read of the frames for both transforms.
template <int S, int IN_MODE, int OUT_MODE, int FRC = 0, int FCC = 0, int NGRP = kDenseTcGroups>
__global__ void __launch_bounds__((4 * NGRP + 3) * 32, 1)
    dense_tc_kernel(const __grid_constant__ CUtensorMap in_map,
                    const __grid_constant__ CUtensorMap out_map, const __grid_constant__ Geom geom,
                    const __grid_constant__ DenseTcParams prm,
                    const __grid_constant__ CUtensorMap adj_map,
                    const __grid_constant__ KParams<float, 32, 32, FRC, FCC> kp) {
  constexpr int NTHR = (4 * NGRP + 3) * 32;
  constexpr bool FUSED = FRC != 0;
  static_assert(!FUSED || (IN_MODE == MODE_FRAME4 && OUT_MODE == MODE_LINEAR),
                "the fused adjusted + exact path reads frames as one-box super-tiles");
  using RowOp = AxisOp<float, 32, FRC>;
  using ColOp = AxisOp<float, 32, FCC>;
  static_assert(!FUSED || (!RowOp::kDense && !ColOp::kDense), "fused ops are the fast paths");
  static_assert(NGRP * 128 <= 512, "TMEM columns");
  // every use of ring stage s then belongs to the same group (tiles k = g mod NGRP,
  // stage k mod S), which waited the stage's previous phase itself: the parity
  // waits on full[s] are exact (shared stages need the hand-off of ring_kernel)
  static_assert(S % NGRP == 0, "ring stages per epilogue group");
  using L = TileLayout<float, 32, 32, 4>;  // 128 rows x 128 B, SW128
  static_assert(L::TILEB == 16384 && L::STAGEB == 16384, "4 blocks of 32x32 fp32");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stages = smem;                     // S x 16 KB: X tiles as loaded
  uint8_t* gtile = smem + S * 16384;          // NGRP x 16 KB: W transpose / Y staging
  uint8_t* bmat = gtile + NGRP * 16384;       // 4 x 4 KB: Dv hi/lo, Dh hi/lo (32 rows)
  uint8_t* dv_hi = bmat;
  uint8_t* dv_lo = bmat + 4096;
  uint8_t* dh_hi = bmat + 8192;
  uint8_t* dh_lo = bmat + 12288;
  uint64_t* full = reinterpret_cast<uint64_t*>(bmat + 16384);
  uint64_t* empty = full + S;
  uint64_t* a1_ready = empty + S;  // per group
  uint64_t* d1_done = a1_ready + NGRP;
  uint64_t* a2_ready = d1_done + NGRP;
  uint64_t* d2_done = a2_ready + NGRP;
  int64_t* tile_id = reinterpret_cast<int64_t*>(d2_done + NGRP);  // per ring stage; -1 = end
  // per group: the tile index of its end marker (set before its ready arrivals)
  volatile int64_t* mma_end = tile_id + S;
  double* red = reinterpret_cast<double*>(tile_id + S + NGRP);  // NGRP x 4 warps x 4 (fused)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red + NGRP * 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // constant B operands: Dv, Dh split into tf32 hi / lo, K-major SW128 (32 rows)
  for (int e = tid; e < 1024; e += NTHR) {
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
      mbar_init(&empty[s], 1);
    }
    for (int g = 0; g < NGRP; ++g) {
      mbar_init(&a1_ready[g], 1);
      mbar_init(&d1_done[g], 1);
      mbar_init(&a2_ready[g], 1);
      mbar_init(&d2_done[g], 1);
    }
    for (int g = 0; g < NGRP; ++g) mma_end[g] = INT64_MAX;
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");  // all of TMEM (one CTA per SM; NGRP x 128 columns used)
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (prm.trace && tid == 0 && blockIdx.x < kTcTraceCtas)
    prm.trace[kTcTraceTiles * kTcTraceEv + 2 * blockIdx.x] = globaltimer();

  // everything above overlaps the previous kernel's tail (programmatic launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t ntiles = geom.ntiles;

  if (warp == 4 * NGRP) {
    // ---------------- TMA producer; chunks of CH tiles: blockIdx.x, then from a
    // global counter, the next chunk's atomic in flight while this one loads
    if (lane == 0) {
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
          const int nb = IN_MODE == MODE_FRAME4 ? 4 : tile_blocks<4, IN_MODE>(t, geom);
          mbar_arrive_expect_tx(&full[s], 4096 * nb);
          tc_tile_io<IN_MODE>(true, stages + s * 16384, &in_map, &full[s], t, geom);
        }
        chunk = gridDim.x + static_cast<int64_t>(nxt);
        if (chunk * CH < ntiles) nxt = atomicAdd(prm.sched, 1ull);
      }
      asm volatile("griddepcontrol.launch_dependents;" :::);
      for (int j = 0; j < NGRP; ++j, ++k) {  // one end marker per epilogue group
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
    const uint32_t dcol = pass1 ? 64 : 96;
    if (lane == 0) {
      for (int64_t k = 0;; ++k) {
        const int g = static_cast<int>(k % NGRP);
        const uint32_t par = static_cast<uint32_t>((k / NGRP) & 1);
        // the dense kernel polls (try_wait's suspend adds latency to a latency-bound
        // pipeline); the fused one is issue-bound and blocks instead, returning the
        // issue slots of the SM sub-partitions it shares with epilogue warps
        if constexpr (FUSED) {
          mbar_wait(&ready[g], par);
        } else {
          while (!mbar_test(&ready[g], par)) {
            if (prm.spin_ns > 0) __nanosleep(prm.spin_ns);
          }
        }
        // group g met its end marker at tile index k: its earlier arrivals are all
        // consumed (it finished tile k - NGRP, both passes, before reaching it)
        if (k >= mma_end[g]) break;
        if (pass1 && prm.trace && blockIdx.x == 0 && k < kTcTraceTiles)
          prm.trace[k * kTcTraceEv + 7] = clock64();
        tc::fence_after();
        tc::gemm3_ts(tmem + 128 * g + dcol, tmem + 128 * g, bhi, blo);
        tc::commit(&done[g]);
      }
    }
  } else {
    // ---------------- epilogue groups
    const int g = warp >> 2;
    const uint32_t b = warp & 3;  // block of the super-tile = TMEM lane quadrant
    const uint32_t lane_addr = (b * 32) << 16;
    const bool leader = b == 0 && lane == 0;
    uint8_t* gt = gtile + g * 16384;
    const uint32_t ta = tmem + 128 * g + lane_addr;  // this lane's A / D1 / D2 columns
    auto group_bar = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory"); };
    // fused: per-thread error sums of the current frame, flushed (group-reduced,
    // one fp64 atomic per value) when the frame changes and at the end
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int acc_f = -1;
    auto flush = [&]() {
      if (acc_f >= 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double a = acc[i];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
          if (lane == 0) red[(g * 4 + b) * 4 + i] = a;
        }
        group_bar();
        if (b == 0 && lane < 4)
          atomicAdd(prm.err + 4 * acc_f + lane, red[(g * 4 + 0) * 4 + lane] + red[(g * 4 + 1) * 4 + lane] +
                                                    red[(g * 4 + 2) * 4 + lane] + red[(g * 4 + 3) * 4 + lane]);
        group_bar();
      }
      acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
    };
    int prev_s = -1;  // fused: ring stage still held by the previous tile
    const bool tr = prm.trace && blockIdx.x == 0 && leader;
    auto ev = [&](int64_t k, int e) {
      if (tr && k < kTcTraceTiles) prm.trace[k * kTcTraceEv + e] = clock64();
    };
    for (int64_t k = g;; k += NGRP) {
      const int s = static_cast<int>(k % S);
      const uint32_t gp = static_cast<uint32_t>((k / NGRP) & 1);  // this group's use parity
      uint8_t* x = stages + s * 16384;
      uint32_t v[32];
      // pass-1 A: column j = lane of block b, A[(b,j)][i] = X_b[i][j]
      ev(k, 0);
      mbar_wait(&full[s], static_cast<uint32_t>((k / S) & 1));
      const int64_t t = tile_id[s];
      if constexpr (FUSED) {
        // the previous tile's stage carried its adjusted output: free it once both
        // of that tile's stores have read shared memory
        if (leader && prev_s >= 0) {
          bulk_wait_read<0>();
          mbar_arrive(&empty[prev_s]);
        }
        prev_s = s;
      }
      if (t < 0) {  // end marker: release the MMA issuers waiting for tile k
        if (leader) {
          mma_end[g] = k;
          mbar_arrive(&a1_ready[g]);
          mbar_arrive(&a2_ready[g]);
        }
        break;
      }
      ev(k, 1);
#pragma unroll
      for (int i = 0; i < 32; ++i)
        v[i] = *reinterpret_cast<const uint32_t*>(x + tc::sw(tc_row<IN_MODE>(b, i), lane));
      tc::st_split(ta, v);
      tc::wait_st();
      if (leader) bulk_wait_read<0>();  // Y(k - NGRP) has left the group tile
      tc::fence_before();
      group_bar();
      if (leader) {
        if constexpr (!FUSED) mbar_arrive(&empty[s]);  // fused: the stage is still needed
        mbar_arrive(&a1_ready[g]);
      }
      // fused: the adjusted transform in place on the interleaved tile, its row
      // pass overlapping MMA pass 1 and its column pass overlapping pass 2 (all 4
      // warps, scalar lanes: a thread owns one row, then one column)
      constexpr int GSQ = RowOp::kGainSq * ColOp::kGainSq;
      const int gl = static_cast<int>(b) * 32 + lane;
      if constexpr (FUSED)
        row_pass<float, 32, 32, 4, FRC, ColOp::kIdentity ? GSQ : 1, false, 128>(x, gl, kp.row,
                                                                               nullptr);
      ev(k, 2);
      // W_b = Dv X_b: lane j holds column j; transpose through this warp's 4 KB
      mbar_wait(&d1_done[g], gp);
      tc::fence_after();
      ev(k, 3);
      tc::ld32(ta + 64, v);
      // Fused: from here on TMEM lane rho = 32 b + lane stands for the row of the INTERLEAVED
      // tile (block rho & 3, block row rho >> 2), the layout of the adjusted tile in the ring
      // stage, so the error pass below reads its Y_a row -- and stages its Y_e row -- at
      // consecutive tile rows per lane (conflict-free; with lane = block row the 8 lanes of
      // an LDS.128 phase hit 2 swizzle columns: 16 wavefronts instead of 4, a quarter of
      // the kernel's shared-memory traffic).  The W transpose therefore goes through the
      // whole group tile (rows 4 r + b) and a group barrier instead of a per-warp tile.
      constexpr bool IL = FUSED;
#pragma unroll
      for (int r = 0; r < 32; ++r)
        *reinterpret_cast<uint32_t*>(gt + tc::sw(IL ? r * 4 + b : b * 32 + r, lane)) = v[r];
      if constexpr (IL)
        group_bar();
      else
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
      if constexpr (FUSED) {  // (the barrier above also closed the row pass)
        col_pass<float, 32, 32, 4, FCC, GSQ, false, 128, true, true>(x, gl, kp.col, nullptr);
        fence_proxy_async_smem();
        group_bar();
        if (leader) {
          tma_store_3d(&adj_map, x, 0, static_cast<int>(4 * t), 0);
          bulk_commit();
        }
      }
      ev(k, 4);
      // Y_b rows from TMEM into the group tile, TMA store
      mbar_wait(&d2_done[g], gp);
      tc::fence_after();
      ev(k, 5);
      tc::ld32(ta + 96, v);
      if constexpr (FUSED) {
        // approximation error of this row: adjusted (stage) vs exact (TMEM)
        float d2 = 0.f, e2 = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 a = *reinterpret_cast<const float4*>(x + tc::sw(gl, q * 4));
          const float ya[4] = {a.x, a.y, a.z, a.w};
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
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint4*>(gt + tc::sw(FUSED ? gl : tc_row<OUT_MODE>(b, lane), q * 4)) =
            make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      fence_proxy_async_smem();
      tc::fence_before();
      group_bar();
      if (leader) {
        if constexpr (FUSED)  // interleaved tile -> block-major memory (out_map: LINEAR_IL view)
          tma_store_3d(&out_map, gt, 0, static_cast<int>(4 * t), 0);
        else
          tc_tile_io<OUT_MODE>(false, gt, &out_map, nullptr, t, geom);
        bulk_commit();
      }
      ev(k, 6);
    }
    if constexpr (FUSED) flush();
    if (leader) bulk_wait_all();
  }
  tc::fence_before();
  __syncthreads();
  if (prm.trace && tid == 0 && blockIdx.x < kTcTraceCtas)
    prm.trace[kTcTraceTiles * kTcTraceEv + 2 * blockIdx.x + 1] = globaltimer();
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

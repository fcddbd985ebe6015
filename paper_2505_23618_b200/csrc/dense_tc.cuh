// dense_tc.cuh -- the dense comparison path on the 5th-generation tensor cores.
//
// Y_b = Dv X_b Dh^T for 32x32 fp32 blocks (the exact DST-7 / DCT-8 of config 5,
// the naive five-transform encoder baseline, Table 1's full-matrix column), as
// two tcgen05.mma (kind::tf32) GEMMs per super-tile of 4 blocks, in 3xTF32
// (a = a_hi + a_lo; a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi: fp32-level error).
//
//   pass 1  D1[(b,i)][n] = sum_k X_b[i][k] Dh[n][k]        M=128 (4 blocks x 32 rows), N=32, K=32
//   pass 2  D2[(b,n)][j] = sum_i Z_b[i][n] Dv[j][i]         (Z_b^T as the A operand)
//   Y_b[j][n] = D2[(b,n)][j]
//
// Operands are K-major 128-byte-swizzled smem tiles: the TMA-loaded block tile
// (P=4 blocks = 128 rows x 128 B) IS the pass-1 A operand.  Accumulators live
// in TMEM (2 x 32 columns); each of the 128 threads owns one TMEM lane and
// moves its row with tcgen05.ld, writing the transposed operand / output tile.
// One elected thread issues the MMAs; completion is tcgen05.commit -> mbarrier.
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
};

// S-stage TMA ring of 4-block super-tiles; one CTA = 8 warps: warps w and w+4
// share TMEM lane quadrant w%4 (tile rows 32(w%4) ..), each moving 16 of the 32
// columns.
// Three tiles are in flight per CTA (TMEM and `lo` buffers triple-buffered) so
// each tensor-core GEMM hides behind a full phase of thread work:
//   iteration k:  A(k)   split X_k into tf32 hi / lo, issue GEMM1(k)
//                 C(k-2) wait GEMM2(k-2), TMEM -> Y tile, TMA store, refill
//                 B(k-1) wait GEMM1(k-1), TMEM -> Z^T operand, issue GEMM2(k-1)
template <int S, int IN_MODE, int OUT_MODE>
__global__ void __launch_bounds__(256)
    dense_tc_kernel(const __grid_constant__ CUtensorMap in_map,
                    const __grid_constant__ CUtensorMap out_map, const __grid_constant__ Geom geom,
                    const __grid_constant__ DenseTcParams prm) {
  using L = TileLayout<float, 32, 32, 4>;  // 128 rows x 128 B, SW128
  static_assert(L::TILEB == 16384 && L::STAGEB == 16384, "4 blocks of 32x32 fp32");
  static_assert(S >= 4, "a stage is held from A(k) until C(k)");
  constexpr int NSLOT = 3;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stages = smem;                       // S x 16 KB: X tile, then Z^T hi
  uint8_t* lobuf = smem + S * 16384;            // NSLOT x 16 KB: X lo, then Z^T lo, then Y
  uint8_t* bmat = lobuf + NSLOT * 16384;        // 4 x 4 KB: Dh hi/lo, Dv hi/lo (32 rows)
  uint8_t* dh_hi = bmat;
  uint8_t* dh_lo = bmat + 4096;
  uint8_t* dv_hi = bmat + 8192;
  uint8_t* dv_lo = bmat + 12288;
  uint64_t* full = reinterpret_cast<uint64_t*>(bmat + 16384);
  uint64_t* bar1 = full + S;       // GEMM1 done, per slot
  uint64_t* bar2 = bar1 + NSLOT;   // GEMM2 done, per slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar2 + NSLOT);
  const int tid = threadIdx.x, warp = tid >> 5;

  // constant operands: split Dh, Dv into tf32 hi / lo, K-major SW128 (32 rows)
  for (int e = tid; e < 1024; e += 256) {
    const int r = e >> 5, c = e & 31;
    const float h = prm.dh[e], v = prm.dv[e];
    const uint32_t hh = tc::tf32_hi(h), vh = tc::tf32_hi(v);
    *reinterpret_cast<uint32_t*>(dh_hi + tc::sw(r, c)) = hh;
    *reinterpret_cast<float*>(dh_lo + tc::sw(r, c)) = h - __uint_as_float(hh);
    *reinterpret_cast<uint32_t*>(dv_hi + tc::sw(r, c)) = vh;
    *reinterpret_cast<float*>(dv_lo + tc::sw(r, c)) = v - __uint_as_float(vh);
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    for (int j = 0; j < NSLOT; ++j) {
      mbar_init(&bar1[j], 1);
      mbar_init(&bar2[j], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t quad = warp & 3, half = warp >> 2;
  const uint32_t lane_addr = (quad * 32) << 16;
  const uint32_t m = quad * 32 + (tid & 31);  // TMEM lane / tile row owned by this thread
  const uint32_t c0 = half * 16;              // the 16 columns this thread moves

  const int64_t ntiles = geom.ntiles;
  const int64_t mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto tile_of = [&](int64_t k) { return blockIdx.x + k * gridDim.x; };
  if (tid == 0) {
    for (int s = 0; s < S && s < mine; ++s) {
      const int64_t t = tile_of(s);
      const int nb = tile_blocks<4, IN_MODE>(t, geom);
      mbar_arrive_expect_tx(&full[s], 4096 * nb);
      issue_tile_io<float, 32, 32, 4, IN_MODE>(true, stages + s * 16384, &in_map, &full[s], t,
                                               geom, nb);
    }
  }

  for (int64_t k = 0; k < mine + 2; ++k) {
    // ---- A(k): split X_k into tf32 hi (in place) and lo; GEMM1(k)
    if (k < mine) {
      const int slot = static_cast<int>(k % NSLOT);
      uint8_t* x = stages + (k % S) * 16384;
      uint8_t* lo = lobuf + slot * 16384;
      mbar_wait(&full[k % S], static_cast<uint32_t>((k / S) & 1));
      if (tid == 0) bulk_wait_read<0>();  // Y(k-3), stored from this lo buffer, is read
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t o = tc::sw(m, c0 + q * 4);
        const float4 v = *reinterpret_cast<const float4*>(x + o);
        const uint4 h =
            make_uint4(tc::tf32_hi(v.x), tc::tf32_hi(v.y), tc::tf32_hi(v.z), tc::tf32_hi(v.w));
        *reinterpret_cast<uint4*>(x + o) = h;
        *reinterpret_cast<float4*>(lo + o) =
            make_float4(v.x - __uint_as_float(h.x), v.y - __uint_as_float(h.y),
                        v.z - __uint_as_float(h.z), v.w - __uint_as_float(h.w));
      }
      fence_proxy_async_smem();
      tc::fence_before();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        tc::gemm3(tmem + 64 * slot, x, lo, dh_hi, dh_lo);
        tc::commit(&bar1[slot]);
      }
    }
    // ---- C(k-2): Y(k-2) from TMEM, store, refill its stage
    if (k >= 2 && k - 2 < mine) {
      const int64_t kp = k - 2;
      const int ps = static_cast<int>(kp % NSLOT);
      uint8_t* plo = lobuf + ps * 16384;
      mbar_wait(&bar2[ps], static_cast<uint32_t>((kp / NSLOT) & 1));
      tc::fence_after();
      uint32_t y[16];
      tc::ld16(tmem + 64 * ps + 32 + c0 + lane_addr, y);
      const uint32_t b = m >> 5, n = m & 31;  // Y_b[j][n] = D2[(b, n)][j]
#pragma unroll
      for (int j = 0; j < 16; ++j)
        *reinterpret_cast<uint32_t*>(plo + tc::sw(b * 32 + c0 + j, n)) = y[j];
      fence_proxy_async_smem();
      tc::fence_before();
      __syncthreads();
      if (tid == 0) {
        const int64_t tp = tile_of(kp);
        issue_tile_io<float, 32, 32, 4, OUT_MODE>(false, plo, &out_map, nullptr, tp, geom,
                                                  tile_blocks<4, OUT_MODE>(tp, geom));
        bulk_commit();
        // the stage of tile k-2 is free (both its GEMMs have read it): refill S ahead
        const int64_t kn = kp + S;
        if (kn < mine) {
          const int64_t tn = tile_of(kn);
          const int nb = tile_blocks<4, IN_MODE>(tn, geom);
          mbar_arrive_expect_tx(&full[kp % S], 4096 * nb);
          issue_tile_io<float, 32, 32, 4, IN_MODE>(true, stages + (kp % S) * 16384, &in_map,
                                                   &full[kp % S], tn, geom, nb);
        }
      }
    }
    // ---- B(k-1): Z^T operand from TMEM, GEMM2(k-1)
    if (k >= 1 && k - 1 < mine) {
      const int64_t kb = k - 1;
      const int bs = static_cast<int>(kb % NSLOT);
      uint8_t* x = stages + (kb % S) * 16384;
      uint8_t* lo = lobuf + bs * 16384;
      mbar_wait(&bar1[bs], static_cast<uint32_t>((kb / NSLOT) & 1));
      tc::fence_after();
      uint32_t z[16];
      tc::ld16(tmem + 64 * bs + c0 + lane_addr, z);
      const uint32_t b = m >> 5, i = m & 31;  // A2[(b, n)][i] = Z_b[i][n]
#pragma unroll
      for (int nn = 0; nn < 16; ++nn) {
        const float zv = __uint_as_float(z[nn]);
        const uint32_t h = tc::tf32_hi(zv);
        const uint32_t o = tc::sw(b * 32 + c0 + nn, i);
        *reinterpret_cast<uint32_t*>(x + o) = h;
        *reinterpret_cast<float*>(lo + o) = zv - __uint_as_float(h);
      }
      fence_proxy_async_smem();
      tc::fence_before();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        tc::gemm3(tmem + 64 * bs + 32, x, lo, dv_hi, dv_lo);
        tc::commit(&bar2[bs]);
      }
    }
  }
  if (tid == 0) bulk_wait_all();
  tc::fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

}  // namespace dctadj

// roundtrip.cu -- launcher and instantiations of the fused forward + inverse
// kernel (roundtrip.cuh).  Op pairs without an instantiation here run as the
// two separate tile kernels (abi.cu), with identical results.
#include "launch.cuh"
#include "roundtrip.cuh"

namespace dctadj {

template <typename T, int H, int W, int P, int RCF, int CCF, int RCI, int CCI, int NG, int S,
          bool PRF, bool PC, bool PRI, int MINB, bool YSTG, int NW, int CH = 0,
          int MODE = MODE_LINEAR>
int launch_roundtrip(const RtArgs& a) {
  using L = TileLayout<T, H, W, P>;
  using Prm = RtParams<T, W, H, RCF, CCF, RCI, CCI>;
  Geom g{};
  if constexpr (MODE == MODE_GATHER) {
    g.nblocks = a.gather_blocks;
    g.ntiles = (g.nblocks + P - 1) / P;
    g.offsets = a.offsets;
  } else {
    g.ntiles = (a.rows + L::PH - 1) / L::PH;
    g.nblocks = g.ntiles * P;
  }
  if (g.ntiles == 0) return ST_OK;
  if constexpr (MODE == MODE_LINEAR) {
    const size_t bytes = static_cast<size_t>(a.rows) * W * sizeof(T);
    g.early = pdl_early(a.stream, {a.in, bytes}, {a.y, bytes}, {a.xr, bytes}) ? 1 : 0;
  } else {
    pdl_poison(a.stream);
  }
  LaunchArgs la;
  la.rows = a.rows;
  CUtensorMap in_map, y_map, xr_map;
  int rc = make_map<T, H, W, P, MODE>(&in_map, a.in, la);
  if (!rc) rc = make_map<T, H, W, P, MODE>(&y_map, a.y, la);
  if (!rc) rc = make_map<T, H, W, P, MODE>(&xr_map, a.xr, la);
  if (rc) return rc;
  Prm prm;
  std::memset(&prm, 0, sizeof(prm));
  if (AxisOp<T, W, RCF>::NCOEF > 0)
    std::memcpy(prm.f.row.c, a.coef[0], sizeof(T) * AxisOp<T, W, RCF>::NCOEF);
  if (AxisOp<T, H, CCF>::NCOEF > 0)
    std::memcpy(prm.f.col.c, a.coef[1], sizeof(T) * AxisOp<T, H, CCF>::NCOEF);
  if (AxisOp<T, W, RCI>::NCOEF > 0)
    std::memcpy(prm.i.row.c, a.coef[2], sizeof(T) * AxisOp<T, W, RCI>::NCOEF);
  if (AxisOp<T, H, CCI>::NCOEF > 0)
    std::memcpy(prm.i.col.c, a.coef[3], sizeof(T) * AxisOp<T, H, CCI>::NCOEF);
  prm.y = static_cast<T*>(a.y);
  prm.nblk = a.rows / H;

  auto kern =
      roundtrip_kernel<T, H, W, P, RCF, CCF, RCI, CCI, NG, S, PRF, PC, PRI, MINB, YSTG, NW, CH, MODE>;
  const size_t smem = 1024 + static_cast<size_t>(NG) * (YSTG ? S : S + 1) * L::STAGEB + NG * S * 8;
  static std::atomic<int> setup[kMaxDevices];  // per instantiation and device
  const int blocks_per_sm = kernel_blocks_per_sm(kern, NG * NW * 32, smem, setup, "roundtrip_kernel");
  if (!blocks_per_sm) return ST_ERR_CUDA;
  const int64_t want = (g.ntiles + NG - 1) / NG;
  const int64_t cap = static_cast<int64_t>(num_sms_cached()) * blocks_per_sm;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(want < cap ? want : cap));
  cfg.blockDim = dim3(NG * NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, in_map, y_map, xr_map, g, prm);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error("roundtrip_kernel launch: %s", cudaGetErrorString(e));
    return ST_ERR_CUDA;
  }
  return ST_OK;
}

// op codes (butterfly.cuh): stage1 | stage2 << 4 | k << 8
constexpr int kSubF = op_code(ST_DCT2, ST_SUB, 8);      // sub-block post, forward
constexpr int kSubI = op_code(ST_SUB, ST_IDCT2, 8);     // sub-block post, inverse
constexpr int kG7F = op_code(ST_GIVENS2, ST_DST3, 6);    // band-6 pre DST-7, forward
constexpr int kG7I = op_code(ST_IDST3, ST_GIVENS2, 6);   // band-6 pre DST-7, inverse
constexpr int kG8F = op_code(ST_GIVENS2, ST_IDCT2, 6);   // band-6 pre DCT-8 (DCT-3 base)
constexpr int kG8I = op_code(ST_DCT2, ST_GIVENS2, 6);

// TUNE(...) keeps a measured-slower tuning variant in the table only when the
// library is built with DCTADJ_TUNING=1 (tools/gen_instances.py, Makefile).
#ifdef DCTADJ_TUNING
#define TUNE(...) __VA_ARGS__,
#define TUNEC(...) , __VA_ARGS__
#else
#define TUNE(...)
#define TUNEC(...)
#endif
#define RTW(T, DT, H, W, P, RF, CF, RI, CI, NG, S, PRF, PC, PRI, MINB, YSTG, NW, VAR)          \
  {DT, H, W, RF, CF, RI, CI, MODE_LINEAR, VAR,                                                   \
   &launch_roundtrip<T, H, W, P, RF, CF, RI, CI, NG, S, PRF, PC, PRI, MINB, YSTG, NW>}
// mixed-shape gather kernels (config 3): 8 KB super-tiles of one class, 4 warps x (2 + 1)
#define RTGV(H, W, RF, CF, RI, CI, PRI, NG, MINB, VAR)                                            \
  {DT_F32, H, W, RF, CF, RI, CI, MODE_GATHER, VAR,                                               \
   &launch_roundtrip<float, H, W, 2048 / (H * W), RF, CF, RI, CI, NG, 2, true, true, PRI, MINB,    \
                     false, 1, 0, MODE_GATHER>}
// sub-8 post classes: default one-warp CTAs, 8 per SM (956 G coef/s on config 3),
// variants 1-4: 4 warps at 255 registers, 3 warps, 2 warps, 4 warps at 128 (941-944);
// band-6 pre classes: 4 warps at 255 registers with scalar inverse rows (762;
// packed inverse rows 752, 128 registers 735, 2- / 1-warp CTAs 761-764)
#define RTG(H, W, RF, CF, RI, CI, PRI, VAR) RTGV(H, W, RF, CF, RI, CI, PRI, 1, 8, VAR)           \
  TUNEC(RTGV(H, W, RF, CF, RI, CI, PRI, 4, 2, VAR + 1), RTGV(H, W, RF, CF, RI, CI, PRI, 3, 3, VAR + 2), \
       RTGV(H, W, RF, CF, RI, CI, PRI, 2, 4, VAR + 3), RTGV(H, W, RF, CF, RI, CI, PRI, 4, 4, VAR + 4))
#define RTGP(H, W, RF, CF, RI, CI) RTGV(H, W, RF, CF, RI, CI, false, 4, 2, 0)                    \
  TUNEC(RTGV(H, W, RF, CF, RI, CI, true, 4, 4, 1), RTGV(H, W, RF, CF, RI, CI, true, 4, 2, 2),      \
       RTGV(H, W, RF, CF, RI, CI, false, 2, 4, 3), RTGV(H, W, RF, CF, RI, CI, false, 1, 8, 4),     \
       RTGV(H, W, RF, CF, RI, CI, false, 3, 3, 5), RTGV(H, W, RF, CF, RI, CI, true, 3, 3, 6))
#define RT(T, DT, H, W, P, RF, CF, RI, CI, NG, S, PRF, PC, PRI, MINB, YSTG, VAR) \
  RTW(T, DT, H, W, P, RF, CF, RI, CI, NG, S, PRF, PC, PRI, MINB, YSTG, 1, VAR)

// variant 0 = default; DCTADJ_RT_VARIANT=k selects tuning variant k where built
static const RtEntry kRt[] = {
    // 32x32 fp32, sub-block post (config 2): 8 KB super-tiles, 4 warps x (2 + 1) stages,
    // 128-register cap (2 CTAs/SM by shared memory); measured variants in profiles/r01_tuning.md
    RT(float, DT_F32, 32, 32, 2, kSubF, kSubF, kSubI, kSubI, 4, 2, true, true, false, 4, false, 0),
    TUNE(RT(float, DT_F32, 32, 32, 2, kSubF, kSubF, kSubI, kSubI, 4, 2, true, true, false, 2, false, 1),
         RT(float, DT_F32, 32, 32, 2, kSubF, kSubF, kSubI, kSubI, 3, 3, true, true, false, 2, false, 2),
         RT(float, DT_F32, 32, 32, 2, kSubF, kSubF, kSubI, kSubI, 3, 2, true, true, false, 3, false, 3),
         RT(float, DT_F32, 32, 32, 2, kSubF, kSubF, kSubI, kSubI, 2, 2, true, true, false, 4, false, 4),
         RT(float, DT_F32, 32, 32, 2, kSubF, kSubF, kSubI, kSubI, 4, 2, true, true, true, 4, false, 5),
         RT(float, DT_F32, 32, 32, 4, kSubF, kSubF, kSubI, kSubI, 2, 2, true, true, false, 4, false, 6))
    // (L2 evict-first hints on the loads, the stores or both: no change, 137.9-139.1 us)
    // (16 KB super-tiles shared by two warps, 2 groups x (2 + 1): 156.6-160.2 us)
    // (one-warp CTAs, 8 per SM: 140.6 us sub-8 post, 183.7 us band-6 pre -- no gain here)
    // y stored from registers (no staging tile; measured slower: 0.83 vs 0.90)
    TUNE(RT(float, DT_F32, 32, 32, 2, kSubF, kSubF, kSubI, kSubI, 4, 2, true, true, false, 3, true, 7),
         RT(float, DT_F32, 32, 32, 2, kSubF, kSubF, kSubI, kSubI, 2, 2, true, true, false, 6, true, 8))
    // 32x32 fp32, band-6 pre (DST-7 / DCT-8 via the DCT-3 base): scalar inverse rows,
    // 255-register budget (177 us per 65,536 blocks; packed inverse rows 188-193 us,
    // y from registers at 12 warps/SM 177 us, 3 warps 219 us)
    RT(float, DT_F32, 32, 32, 2, kG7F, kG7F, kG7I, kG7I, 4, 2, true, true, false, 2, false, 0),
    RT(float, DT_F32, 32, 32, 2, kG8F, kG8F, kG8I, kG8I, 4, 2, true, true, false, 2, false, 0),
    TUNE(RT(float, DT_F32, 32, 32, 2, kG7F, kG7F, kG7I, kG7I, 4, 2, true, true, true, 2, false, 1),
         RT(float, DT_F32, 32, 32, 2, kG7F, kG7F, kG7I, kG7I, 4, 2, true, true, true, 3, true, 3))
    // 64x64 fp32 (config 4): built as tuning variants only -- measured slower than
    // the two tile kernels (shared memory holds 4-8 warps/SM at 16 KB per block
    // and 3 buffers per group: sub-8 post 0.52-0.62, band-6 pre 0.44 of the copy
    // peak vs 0.95 / 0.72 for the two kernels), so the default is the two-kernel path
    // (y from registers, 6 two-warp groups x 2 stages = 12 warps/SM: post 824 / pre 530
    //  G coef/s against 797 / 600 for the two kernels; 4 groups x 3 stages 750, one-warp
    //  packed groups 697-760; one two-warp group per CTA, 6 CTAs/SM: post 799, pre 572)
    TUNE(RT(float, DT_F32, 64, 64, 1, kSubF, kSubF, kSubI, kSubI, 4, 2, true, true, true, 1, false, 1),
         RTW(float, DT_F32, 64, 64, 1, kSubF, kSubF, kSubI, kSubI, 4, 2, false, false, false, 1, false, 2, 2),
         RTW(float, DT_F32, 64, 64, 1, kG7F, kG7F, kG7I, kG7I, 4, 2, false, false, false, 1, false, 2, 1),
         RTW(float, DT_F32, 64, 64, 1, kSubF, kSubF, kSubI, kSubI, 6, 2, false, false, false, 1, true, 2, 3),
         RTW(float, DT_F32, 64, 64, 1, kG7F, kG7F, kG7I, kG7I, 6, 2, false, false, false, 1, true, 2, 3),
         RTW(float, DT_F32, 64, 64, 1, kG8F, kG8F, kG8I, kG8I, 6, 2, false, false, false, 1, true, 2, 3),
         RTW(float, DT_F32, 64, 64, 1, kG8F, kG8F, kG8I, kG8I, 4, 2, false, false, false, 1, false, 2, 1))
    // config 3 classes: {16,32}^2 shapes, sub-block post (DST-7 / DCT-8 share the ops) and
    // band-6 pre with DST-7 or DCT-8 per axis
    RTG(16, 16, kSubF, kSubF, kSubI, kSubI, false, 0),
    RTG(16, 32, kSubF, kSubF, kSubI, kSubI, false, 0),
    RTG(32, 16, kSubF, kSubF, kSubI, kSubI, false, 0),
    RTG(32, 32, kSubF, kSubF, kSubI, kSubI, false, 0),
#define RTG_PRE(H, W)                                      \
  RTGP(H, W, kG7F, kG7F, kG7I, kG7I), RTGP(H, W, kG7F, kG8F, kG7I, kG8I), \
      RTGP(H, W, kG8F, kG7F, kG8I, kG7I), RTGP(H, W, kG8F, kG8F, kG8I, kG8I)
    RTG_PRE(16, 16),
    RTG_PRE(16, 32),
    RTG_PRE(32, 16),
    RTG_PRE(32, 32),
#undef RTG_PRE
};

#undef TUNE
#undef TUNEC
#undef RT
#undef RTW
#undef RTG
#undef RTGP
#undef RTGV

const RtEntry* find_roundtrip(int dtype, int h, int w, int rcf, int ccf, int rci, int cci,
                              int mode, int variant) {
  const RtEntry* dflt = nullptr;
  for (const RtEntry& e : kRt)
    if (e.dtype == dtype && e.h == h && e.w == w && e.rcf == rcf && e.ccf == ccf &&
        e.rci == rci && e.cci == cci && e.mode == mode) {
      if (e.variant == variant) return &e;
      if (e.variant == 0) dflt = &e;
    }
  return dflt;
}

}  // namespace dctadj

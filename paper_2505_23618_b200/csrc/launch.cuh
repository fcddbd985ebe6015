// launch.cuh -- host-side launcher for one tile_kernel instantiation:
// builds the TMA tensor maps, packs the per-axis coefficients into the kernel
// parameter block (they are read as constant-bank operands by the FMAs), sizes
// a persistent grid, and launches on the caller's stream.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstring>

#include "tile_kernel.cuh"

namespace dctadj {

enum DType : int { DT_F32 = 0, DT_F64 = 1 };

struct LaunchArgs {
  const void* in = nullptr;
  void* out = nullptr;
  // LINEAR side: total rows (nblk * H for 2-D, nvec for 1-D)
  int64_t rows = 0;
  // FRAME side: nframes x frame_h x frame_w samples
  int32_t frames = 0, frame_h = 0, frame_w = 0;
  const void* row_coef = nullptr;  // host, packed AxisOp::Coef of the row op
  const void* col_coef = nullptr;  // host, packed AxisOp::Coef of the column op
  const void* dense_row = nullptr; // device, W x W (row op ST_DENSE)
  const void* dense_col = nullptr; // device, H x H (column op ST_DENSE)
  // GATHER side: `gather_blocks` blocks at element offsets `offsets` (device)
  // of a packed buffer of `rows` x W elements
  const int64_t* offsets = nullptr;
  int64_t gather_blocks = 0;
  cudaStream_t stream = nullptr;
};

// status codes shared with the C-ABI (include/dctadj.h)
enum : int {
  ST_OK = 0,
  ST_ERR_DIMENSION = 1,
  ST_ERR_SHAPE = 2,
  ST_ERR_PATTERN = 3,
  ST_ERR_CONFIG = 4,
  ST_ERR_KIND = 5,
  ST_ERR_CUDA = 6,
  ST_ERR_UNSUPPORTED = 7,
  ST_ERR_VALUE = 8,
};

// implemented in abi.cu
int encode_tensor_map(CUtensorMap* map, int dtype, int rank, const uint64_t* dims,
                      const uint64_t* strides_bytes, const uint32_t* box, int box_row_bytes,
                      void* base);
int num_sms_cached();
// Cross-launch overlap bookkeeping (abi.cu): may a launch reading [in, in + nin)
// and writing the two output ranges skip the entry wait on the previous grid of
// the stream (it overlaps none of the ranges of the launches that may still be
// running there)?  Records the launch either way.  pdl_poison: a launch whose
// ranges are not tracked -- the next launch on the stream waits at entry.
struct ByteRange {
  const void* p;
  size_t n;
};
bool pdl_early(cudaStream_t st, ByteRange in, ByteRange out1, ByteRange out2 = {nullptr, 0});
void pdl_poison(cudaStream_t st);
void set_last_error(const char* fmt, ...);

// One-time launch setup of a kernel on the current device (dynamic shared
// memory limit, max-shared carveout, occupancy query), cached per device in
// the caller's per-instantiation slot array.  Function attributes are per
// device context, so each device of a multi-GPU process configures its own;
// racing first calls both run the (idempotent) setup.  Returns resident CTAs
// per SM (>= 1), or 0 with the error message set.
constexpr int kMaxDevices = 64;
template <typename K>
int kernel_blocks_per_sm(K kern, int threads, size_t smem, std::atomic<int> (&slot)[kMaxDevices],
                         const char* what) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  const int cached = slot[dev].load(std::memory_order_acquire);
  if (cached > 0) return cached;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  int nb = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem);
  if (e != cudaSuccess || nb < 1) {
    set_last_error("%s setup: %s (%d CTAs/SM with %zu B shared memory)", what,
                   cudaGetErrorString(e), nb, smem);
    return 0;
  }
  slot[dev].store(nb, std::memory_order_release);
  return nb;
}

template <typename T, int H, int W, int P, int MODE>
int make_map(CUtensorMap* map, const void* base, const LaunchArgs& a) {
  using L = TileLayout<T, H, W, P>;
  constexpr int dt = sizeof(T) == 4 ? DT_F32 : DT_F64;
  if constexpr (MODE == MODE_LINEAR_IL) {  // (nblk, H, W) as {W, block, row}
    uint64_t dims[3] = {static_cast<uint64_t>(W), static_cast<uint64_t>(a.rows / H),
                        static_cast<uint64_t>(H)};
    uint64_t strides[2] = {static_cast<uint64_t>(H) * W * sizeof(T), static_cast<uint64_t>(W) * sizeof(T)};
    uint32_t box[3] = {static_cast<uint32_t>(W), static_cast<uint32_t>(P), static_cast<uint32_t>(H)};
    return encode_tensor_map(map, dt, 3, dims, strides, box, L::BRB, const_cast<void*>(base));
  } else if constexpr (MODE == MODE_FRAME_IL) {  // {W, block column, frame row, frame}
    uint64_t dims[4] = {static_cast<uint64_t>(W), static_cast<uint64_t>(a.frame_w / W),
                        static_cast<uint64_t>(a.frame_h), static_cast<uint64_t>(a.frames)};
    uint64_t strides[3] = {static_cast<uint64_t>(W) * sizeof(T),
                           static_cast<uint64_t>(a.frame_w) * sizeof(T),
                           static_cast<uint64_t>(a.frame_w) * a.frame_h * sizeof(T)};
    uint32_t box[4] = {static_cast<uint32_t>(W), static_cast<uint32_t>(P), static_cast<uint32_t>(H), 1u};
    return encode_tensor_map(map, dt, 4, dims, strides, box, L::BRB, const_cast<void*>(base));
  } else if constexpr (MODE == MODE_LINEAR || MODE == MODE_GATHER) {
    uint64_t dims[2] = {static_cast<uint64_t>(W), static_cast<uint64_t>(a.rows)};
    uint64_t strides[1] = {static_cast<uint64_t>(W) * sizeof(T)};
    uint32_t box[2] = {static_cast<uint32_t>(L::BW),
                       static_cast<uint32_t>(MODE == MODE_GATHER ? H : L::PH)};
    return encode_tensor_map(map, dt, 2, dims, strides, box, L::BRB, const_cast<void*>(base));
  } else {
    uint64_t dims[3] = {static_cast<uint64_t>(a.frame_w), static_cast<uint64_t>(a.frame_h),
                        static_cast<uint64_t>(a.frames)};
    uint64_t strides[2] = {static_cast<uint64_t>(a.frame_w) * sizeof(T),
                           static_cast<uint64_t>(a.frame_w) * a.frame_h * sizeof(T)};
    uint32_t box[3] = {static_cast<uint32_t>(L::BW), static_cast<uint32_t>(H), 1u};
    return encode_tensor_map(map, dt, 3, dims, strides, box, L::BRB, const_cast<void*>(base));
  }
}

template <typename T, int H, int W, int P, int RC, int CC, bool COL_FIRST, int IN_MODE,
          int OUT_MODE, int NG, int S, bool PAIR_ROW = false, bool PAIR_COL = false, int CH = 0,
          int NW = 1>
int launch_tile(const LaunchArgs& a) {
  using L = TileLayout<T, H, W, P>;
  using RowOp = AxisOp<T, W, RC>;
  using ColOp = AxisOp<T, H, CC>;
  static_assert(S >= 2, "ring needs at least two stages");

  constexpr bool FR = IN_MODE == MODE_FRAME || OUT_MODE == MODE_FRAME ||
                      IN_MODE == MODE_FRAME_IL || OUT_MODE == MODE_FRAME_IL;
  if constexpr (is_il_mode<IN_MODE>()) {
    if ((a.frame_w / W) % P != 0) return ST_ERR_UNSUPPORTED;  // caller falls back to FRAME
  }
  Geom g{};
  if (FR) {
    g.tiles_y = (a.frame_h + H - 1) / H;
    g.tiles_x = a.frame_w / W;
    g.nblocks = static_cast<int64_t>(a.frames) * g.tiles_y * g.tiles_x;
    g.ntiles = (g.nblocks + P - 1) / P;
  } else if (IN_MODE == MODE_GATHER) {
    g.nblocks = a.gather_blocks;
    g.ntiles = (g.nblocks + P - 1) / P;
    g.offsets = a.offsets;
  } else {
    g.ntiles = (a.rows + L::PH - 1) / L::PH;
    g.nblocks = g.ntiles * P;
  }
  if (g.ntiles == 0) return ST_OK;
  g.dense_row = a.dense_row;
  g.dense_col = a.dense_col;
  if constexpr (IN_MODE == MODE_LINEAR && OUT_MODE == MODE_LINEAR) {
    const size_t bytes = static_cast<size_t>(g.ntiles) * L::PH * W * sizeof(T);
    g.early = pdl_early(a.stream, {a.in, bytes}, {a.out, bytes}) ? 1 : 0;
  } else {
    pdl_poison(a.stream);
  }

  // the LINEAR side of a frame launch holds ntiles whole blocks
  LaunchArgs la = a;
  if (FR) la.rows = g.nblocks * H;

  CUtensorMap in_map, out_map;
  int rc = make_map<T, H, W, P, IN_MODE>(&in_map, a.in, la);
  if (rc) return rc;
  rc = make_map<T, H, W, P, OUT_MODE>(&out_map, a.out, la);
  if (rc) return rc;

  KParams<T, W, H, RC, CC> prm;
  std::memset(&prm, 0, sizeof(prm));
  if (RowOp::NCOEF > 0) std::memcpy(prm.row.c, a.row_coef, sizeof(T) * RowOp::NCOEF);
  if (ColOp::NCOEF > 0) std::memcpy(prm.col.c, a.col_coef, sizeof(T) * ColOp::NCOEF);

  if constexpr ((CH & 8) != 0) {  // shared-ring kernel: NG compute warps + a producer, S stages
    static_assert(P == 1 && IN_MODE == MODE_LINEAR && OUT_MODE == MODE_LINEAR,
                  "the ring kernel moves whole LINEAR blocks");
    auto kern = ring_kernel<T, H, W, RC, CC, COL_FIRST, NG, S>;
    const size_t smem = 1024 + static_cast<size_t>(S) * L::STAGEB + 2 * S * 8;
    static std::atomic<int> setup[kMaxDevices];
    if (!kernel_blocks_per_sm(kern, (NG + 1) * 32, smem, setup, "ring_kernel")) return ST_ERR_CUDA;
    const int64_t cap = num_sms_cached();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(g.ntiles < cap ? g.ntiles : cap));
    cfg.blockDim = dim3((NG + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = a.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, in_map, out_map, g, prm);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_last_error("ring_kernel launch: %s", cudaGetErrorString(e));
      return ST_ERR_CUDA;
    }
    return ST_OK;
  } else {
  auto kern = tile_kernel<T, H, W, P, RC, CC, COL_FIRST, IN_MODE, OUT_MODE, NG, S, PAIR_ROW, PAIR_COL, CH, NW>;
  const size_t dense_bytes =
      sizeof(T) * ((RowOp::kDense ? W * W : 0) + (ColOp::kDense ? H * H : 0));
  const size_t smem = 1024 + static_cast<size_t>(NG) * S * L::STAGEB + NG * S * 8 + dense_bytes;

  static std::atomic<int> setup[kMaxDevices];  // per instantiation and device
  const int blocks_per_sm = kernel_blocks_per_sm(kern, NG * NW * 32, smem, setup, "tile_kernel");
  if (!blocks_per_sm) return ST_ERR_CUDA;
  const int64_t want = (g.ntiles + NG - 1) / NG;
  const int64_t cap = static_cast<int64_t>(num_sms_cached()) * blocks_per_sm;
  const int grid = static_cast<int>(want < cap ? want : cap);

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NG * NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, in_map, out_map, g, prm);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error("tile_kernel launch: %s", cudaGetErrorString(e));
    return ST_ERR_CUDA;
  }
  return ST_OK;
  }
}

}  // namespace dctadj

// abi.cu -- the C-ABI (include/dctadj.h): validation with the reference's error
// semantics, per-axis planning (stage codes + packed coefficients), kernel
// dispatch over the generated instantiation table, TMA tensor-map encoding, and
// the pipelined host-buffer entry points.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <vector>

#include "../../include/dctadj.h"
#include "dense_tc.cuh"
#include "dense_tc64.cuh"
#include "enc5.cuh"
#ifdef DCTADJ_TUNING
#include "frames_exact.cuh"
#endif
#include "givens_pack.h"
#include "launch.cuh"
#include "roundtrip.cuh"

namespace dctadj {

struct KernelEntry {
  int dtype, h, w, rc, cc, col_first, in_mode, out_mode, variant;
  int (*fn)(const LaunchArgs&);
};

#include "gen/registry.inc"

static_assert(ST_ERR_DIMENSION == DCTADJ_ERR_DIMENSION && ST_ERR_VALUE == DCTADJ_ERR_VALUE,
              "status codes drifted from include/dctadj.h");

static thread_local char g_err[512] = "";

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define DA_CUDA(call)                                                           \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      return fail(ST_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_));        \
  } while (0)

// ------------------------------------------------------------- tensor maps
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

int encode_tensor_map(CUtensorMap* map, int dtype, int rank, const uint64_t* dims,
                      const uint64_t* strides_bytes, const uint32_t* box, int box_row_bytes,
                      void* base) {
  if (reinterpret_cast<uintptr_t>(base) & 15)
    return fail(ST_ERR_VALUE, "data pointer %p is not 16-byte aligned (TMA requirement)", base);
  EncodeFn fn = get_encode();
  if (!fn) return fail(ST_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i + 1 < rank) s[i] = strides_bytes[i];
  }
  CUtensorMapSwizzle swz = box_row_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                           : box_row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                           : box_row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                 : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = fn(map, dtype == DT_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                  rank, base, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): rank %d dims %llu x %llu",
                (int)r, rank, (unsigned long long)d[0], (unsigned long long)d[1]);
  return ST_OK;
}

int num_sms_cached() {
  static std::atomic<int> cache[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = n > 0 ? n : 1;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// DCTADJ_VARIANT=k selects tuning variant k where one was built (tools/gen_instances.py
// EXPERIMENT); variant 0 is the default build of every configuration.
static int tuning_variant() {
  static int v = [] {
    const char* s = std::getenv("DCTADJ_VARIANT");
    return s ? std::atoi(s) : 0;
  }();
  return v;
}

// DCTADJ_TRACE=1 prints every kernel selection to stderr (diagnostics)
static bool trace_on() {
  static bool v = std::getenv("DCTADJ_TRACE") != nullptr;
  return v;
}

static const KernelEntry* find_kernel(int dtype, int h, int w, int rc, int cc, int col_first,
                                      int in_mode, int out_mode) {
  const KernelEntry* dflt = nullptr;
  const KernelEntry* hit = nullptr;
  const int want = tuning_variant();
  for (const KernelEntry& e : kRegistry)
    if (e.dtype == dtype && e.h == h && e.w == w && e.rc == rc && e.cc == cc &&
        e.col_first == col_first && e.in_mode == in_mode && e.out_mode == out_mode) {
      if (e.variant == want) hit = &e;
      if (e.variant == 0) dflt = &e;
    }
  if (!hit) hit = dflt;
  if (trace_on())
    std::fprintf(stderr, "[dctadj] dtype=%d %dx%d rc=0x%x cc=0x%x col_first=%d mode=%d->%d: %s (variant %d)\n",
                 dtype, h, w, rc, cc, col_first, in_mode, out_mode, hit ? "found" : "MISSING",
                 hit ? hit->variant : -1);
  return hit;
}

// ------------------------------------------------------------- axis planning
static bool fast_size(int n) { return n == 4 || n == 8 || n == 16 || n == 32 || n == 64; }

// exact base matrices from the closed forms (reference transforms.py:78-120)
static void base_matrix(int base, int n, std::vector<double>& m) {
  m.assign(static_cast<size_t>(n) * n, 0.0);
  std::vector<double> c2(static_cast<size_t>(n) * n);
  const double pi = 3.141592653589793238462643383279502884;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) {
      double v = std::cos(pi * k * (2 * j + 1) / (2.0 * n)) * std::sqrt(2.0 / n);
      if (k == 0) v *= 0.7071067811865476;
      c2[k * n + j] = v;
    }
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < n; ++j) {
      if (base == DCTADJ_BASE_DCT2)
        m[r * n + j] = c2[r * n + j];
      else if (base == DCTADJ_BASE_DCT3)
        m[r * n + j] = c2[j * n + r];
      else  // DST3 = S * DCT2^T * R: (r, j) -> (-1)^r DCT2[n-1-j][r]
        m[r * n + j] = ((r & 1) ? -1.0 : 1.0) * c2[(n - 1 - j) * n + r];
    }
}

struct AxisPlan {
  int n = 0;
  int code = 0;
  int gain_sq = 1;
  std::vector<double> coef;   // packed band / sub-block coefficients (fp64)
  // the same for fp64 kernels where their base form differs from fp32's (a Givens
  // stage behind a deferred-scale base, butterfly.cuh deferred_policy); else empty
  std::vector<double> coef64;
  std::vector<double> dense;  // n x n for ST_DENSE
};

static int validate_axis(const dctadj_axis* ax) {
  if (!ax) return fail(ST_ERR_VALUE, "axis descriptor is NULL");
  if (!fast_size(ax->n))
    return fail(ST_ERR_DIMENSION, "fast transforms support sizes (4, 8, 16, 32, 64), got %d",
                ax->n);
  if (ax->base < DCTADJ_BASE_DCT2 || ax->base > DCTADJ_BASE_DCT3)
    return fail(ST_ERR_CONFIG, "no fast path for base transform %d; use dct2, dst3 or dct3",
                ax->base);
  if (ax->adj < DCTADJ_ADJ_NONE || ax->adj > DCTADJ_ADJ_DENSE)
    return fail(ST_ERR_PATTERN, "unknown adjustment kind %d", ax->adj);
  if (ax->side != DCTADJ_SIDE_PRE && ax->side != DCTADJ_SIDE_POST)
    return fail(ST_ERR_CONFIG, "unknown adjustment side %d", ax->side);
  if (ax->adj != DCTADJ_ADJ_NONE && !ax->mat)
    return fail(ST_ERR_VALUE, "adjustment matrix pointer is NULL");
  if (ax->adj == DCTADJ_ADJ_BAND && (ax->taps < 1 || ax->taps > ax->n))
    return fail(ST_ERR_PATTERN, "band taps must be in 1..%d, got %d", ax->n, ax->taps);
  if (ax->adj == DCTADJ_ADJ_SUBBLOCK && (ax->order < 1 || ax->order > ax->n))
    return fail(ST_ERR_PATTERN, "sub-block order must be in 1..%d, got %d", ax->n, ax->order);
  if (ax->ngivens < 0 || (ax->ngivens > 0 && !ax->givens))
    return fail(ST_ERR_VALUE, "bad Givens schedule (%d angles)", ax->ngivens);
  return ST_OK;
}

static double mat_at(const dctadj_axis* ax, bool transpose, int r, int j) {
  const int n = ax->n;
  return transpose ? ax->mat[j * n + r] : ax->mat[r * n + j];
}

// The whole axis as one dense matrix (forward H = B*A or C*B; inverse H^T).
static void composite_dense_uncached(const dctadj_axis* ax, bool inverse, std::vector<double>& out);

// The composite (an O(n^3) host product plus n^2 cosines: ~150 us at n = 64) is
// memoised by the axis contents, so repeated calls with the same transform cost
// a comparison of the n x n input matrix.
struct CompositeKey {
  int n, base, adj, side, taps, order, inverse;
  std::vector<double> mat;
  bool operator==(const CompositeKey& o) const {
    return n == o.n && base == o.base && adj == o.adj && side == o.side && taps == o.taps &&
           order == o.order && inverse == o.inverse && mat == o.mat;
  }
};
static void composite_dense(const dctadj_axis* ax, bool inverse, std::vector<double>& out) {
  static std::mutex mu;
  static std::vector<std::pair<CompositeKey, std::vector<double>>> memo;
  CompositeKey key{ax->n, ax->base, ax->adj, ax->side, ax->taps, ax->order, inverse ? 1 : 0, {}};
  if (ax->mat) key.mat.assign(ax->mat, ax->mat + static_cast<size_t>(ax->n) * ax->n);
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : memo)
      if (e.first == key) {
        out = e.second;
        return;
      }
  }
  composite_dense_uncached(ax, inverse, out);
  std::lock_guard<std::mutex> lk(mu);
  if (memo.size() >= 32) memo.erase(memo.begin());
  memo.emplace_back(std::move(key), out);
}

static void composite_dense_uncached(const dctadj_axis* ax, bool inverse, std::vector<double>& out) {
  const int n = ax->n;
  std::vector<double> b, a(static_cast<size_t>(n) * n, 0.0), h(static_cast<size_t>(n) * n, 0.0);
  base_matrix(ax->base, n, b);
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < n; ++j) {
      double v;
      if (ax->adj == DCTADJ_ADJ_NONE) {
        v = (r == j) ? 1.0 : 0.0;
      } else if (ax->adj == DCTADJ_ADJ_BAND) {  // only in-band entries are read (_fastcore.pyx:261-272)
        v = (std::abs(r - j) < ax->taps) ? ax->mat[r * n + j] : 0.0;
      } else if (ax->adj == DCTADJ_ADJ_SUBBLOCK) {  // identity outside the leading block
        v = (r < ax->order && j < ax->order) ? ax->mat[r * n + j] : (r == j ? 1.0 : 0.0);
      } else {
        v = ax->mat[r * n + j];
      }
      a[r * n + j] = v;
    }
  const bool pre = ax->side == DCTADJ_SIDE_PRE;
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += pre ? b[r * n + k] * a[k * n + j] : a[r * n + k] * b[k * n + j];
      h[r * n + j] = acc;
    }
  out.assign(static_cast<size_t>(n) * n, 0.0);
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < n; ++j) out[r * n + j] = inverse ? h[j * n + r] : h[r * n + j];
}

static void pack_band(const dctadj_axis* ax, bool transpose, int k, std::vector<double>& c) {
  const int n = ax->n, d = 2 * k - 1;
  c.assign(static_cast<size_t>(n) * d, 0.0);
  for (int r = 0; r < n; ++r)
    for (int t = 0; t < d; ++t) {
      const int j = r - (k - 1) + t;
      if (j >= 0 && j < n && std::abs(r - j) < ax->taps) c[r * d + t] = mat_at(ax, transpose, r, j);
    }
}

// scaled-rotation packing of a Givens schedule: givens_pack.h (host only, shared with
// the CPU unit test of the butterflies)
static bool pack_givens2(const dctadj_axis* ax, bool inverse, double gain, int base_before,
                         std::vector<double>& c) {
  return pack_givens2(ax->n, ax->taps, ax->givens, inverse, gain, base_before, c);
}

static void pack_sub(const dctadj_axis* ax, bool transpose, int k, std::vector<double>& c) {
  c.assign(static_cast<size_t>(k) * k, 0.0);
  for (int r = 0; r < k; ++r)
    for (int j = 0; j < k; ++j) c[r * k + j] = mat_at(ax, transpose, r, j);
}

// Stage codes for one axis.  force_dense: plan the dense composite instead.
static int plan_axis(const dctadj_axis* ax, bool inverse, bool force_dense, AxisPlan* p) {
  int rc = validate_axis(ax);
  if (rc) return rc;
  p->n = ax->n;
  p->coef.clear();
  p->dense.clear();
  const int bf = ax->base == DCTADJ_BASE_DCT2 ? ST_DCT2 : ax->base == DCTADJ_BASE_DST3 ? ST_DST3 : ST_IDCT2;
  const int bi = ax->base == DCTADJ_BASE_DCT2 ? ST_IDCT2 : ax->base == DCTADJ_BASE_DST3 ? ST_IDST3 : ST_DCT2;
  const int base = inverse ? bi : bf;
  int adj_stage = ST_NONE, k = 0;
  // a band with its Givens schedule: scaled rotations (2 FMAs each); the stage
  // trails the base for the inverse PRE / forward POST order, where the base's
  // gain sqrt(n) is folded into the final scales
  const bool adj_first = (ax->side == DCTADJ_SIDE_PRE) != inverse;
  const double ggain = adj_first ? 1.0 : 1.0 / std::sqrt(static_cast<double>(ax->n));
  const bool defer32 = !adj_first && deferred_policy(false, ax->n);
  const bool defer64 = !adj_first && deferred_policy(true, ax->n);
  p->coef64.clear();
  if (ax->adj == DCTADJ_ADJ_BAND && (ax->taps == 4 || ax->taps == 6) && ax->givens &&
      ax->ngivens == givens_rots(ax->n, ax->taps) && !force_dense &&
      pack_givens2(ax, inverse, ggain, defer32 ? base : ST_NONE, p->coef)) {
    if (defer64 != defer32) pack_givens2(ax, inverse, ggain, defer64 ? base : ST_NONE, p->coef64);
    adj_stage = ST_GIVENS2;
    k = ax->taps;
  } else if (ax->adj == DCTADJ_ADJ_BAND && (ax->taps == 4 || ax->taps == 6)) {
    adj_stage = ST_BAND;
    k = ax->taps;
    pack_band(ax, inverse, k, p->coef);
  } else if (ax->adj == DCTADJ_ADJ_SUBBLOCK && ax->order == 8) {
    adj_stage = ST_SUB;
    k = 8;
    pack_sub(ax, inverse, k, p->coef);
    // behind a deferred-scale DCT-2 (butterfly.cuh AxisOp::kDeferredSub) the block acts on
    // held values: fold their scales into its columns (fp32 kernels; fp64 keeps the block)
    if (!adj_first && base == ST_DCT2 && !force_dense && (defer32 || defer64)) {
      std::vector<double> folded = p->coef;
      fold_sub_scales(ax->n, k, folded);
      if (defer64 != defer32) p->coef64 = defer64 ? folded : p->coef;
      if (defer32) p->coef = folded;
    }
  } else if (ax->adj != DCTADJ_ADJ_NONE) {
    force_dense = true;
  }
  if (force_dense) {
    composite_dense(ax, inverse, p->dense);
    p->code = op_code(ST_DENSE);
    p->gain_sq = 1;
    p->coef.clear();
    p->coef64.clear();
    return ST_OK;
  }
  p->gain_sq = ax->n;
  if (adj_stage == ST_NONE)
    p->code = op_code(base);
  else if (adj_first)  // fwd PRE or inv POST: adjustment first
    p->code = op_code(adj_stage, base, k);
  else
    p->code = op_code(base, adj_stage, k);
  if (adj_stage == ST_GIVENS2 && !adj_first) p->gain_sq = 1;
  return ST_OK;
}

static size_t dt_size(int dtype) { return dtype == DT_F32 ? 4 : 8; }

static std::vector<unsigned char> to_dtype(const std::vector<double>& v, int dtype);
// an axis plan's coefficients for kernels of element type `dtype`
static std::vector<unsigned char> plan_coef(const AxisPlan& p, int dtype) {
  return to_dtype(dtype == DT_F64 && !p.coef64.empty() ? p.coef64 : p.coef, dtype);
}

// fp64 host coefficients -> the kernel's element type
static std::vector<unsigned char> to_dtype(const std::vector<double>& v, int dtype) {
  std::vector<unsigned char> out(v.size() * dt_size(dtype) + 8);
  if (dtype == DT_F32) {
    float* f = reinterpret_cast<float*>(out.data());
    for (size_t i = 0; i < v.size(); ++i) f[i] = static_cast<float>(v[i]);
  } else {
    std::memcpy(out.data(), v.data(), v.size() * sizeof(double));
  }
  return out;
}

// Dense matrices (composites, the exact comparison transforms) are cached on the
// device by content: a call stream-orders nothing and allocates nothing once the
// matrix has been seen.  A miss uploads synchronously, so the copy is visible to
// every stream.  upload_dense PINS the entry it returns; the caller unpins it
// (release_dense, done by ~Launch / Launch::reset) once its kernels are enqueued,
// so an entry is never evicted between lookup and launch -- by this call's own
// second upload or by another thread.  When the cache is full the least
// recently used unpinned entry of this device is freed after a device-wide
// synchronisation (kernels enqueued earlier may still read it); if every entry
// is pinned the cache grows instead.
struct DenseCacheEntry {
  int device, dtype;
  std::vector<double> m;
  void* ptr;
  int pins;
  uint64_t last_use;
};
static std::mutex g_dense_mu;
static std::vector<DenseCacheEntry> g_dense_cache;
static uint64_t g_dense_tick = 0;
static constexpr size_t kDenseCacheSlots = 64;

static int upload_dense(const AxisPlan& p, int dtype, cudaStream_t st, void** dev) {
  (void)st;
  *dev = nullptr;
  if (p.dense.empty()) return ST_OK;
  int device = 0;
  DA_CUDA(cudaGetDevice(&device));
  std::lock_guard<std::mutex> lk(g_dense_mu);
  for (auto& e : g_dense_cache)
    if (e.device == device && e.dtype == dtype && e.m == p.dense) {
      ++e.pins;
      e.last_use = ++g_dense_tick;
      *dev = e.ptr;
      return ST_OK;
    }
  if (g_dense_cache.size() >= kDenseCacheSlots) {
    size_t victim = g_dense_cache.size();
    for (size_t i = 0; i < g_dense_cache.size(); ++i) {
      const auto& e = g_dense_cache[i];
      if (e.pins == 0 && e.device == device &&
          (victim == g_dense_cache.size() || e.last_use < g_dense_cache[victim].last_use))
        victim = i;
    }
    if (victim < g_dense_cache.size()) {
      DA_CUDA(cudaDeviceSynchronize());  // kernels enqueued before may still read it
      DA_CUDA(cudaFree(g_dense_cache[victim].ptr));
      g_dense_cache.erase(g_dense_cache.begin() + static_cast<std::ptrdiff_t>(victim));
    }
  }
  std::vector<unsigned char> host = to_dtype(p.dense, dtype);
  void* ptr = nullptr;
  DA_CUDA(cudaMalloc(&ptr, host.size()));
  DA_CUDA(cudaMemcpy(ptr, host.data(), host.size(), cudaMemcpyHostToDevice));
  g_dense_cache.push_back({device, dtype, p.dense, ptr, 1, ++g_dense_tick});
  *dev = ptr;
  return ST_OK;
}

// unpin an entry returned by upload_dense (NULL: no-op)
static void release_dense(void* ptr) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lk(g_dense_mu);
  for (auto& e : g_dense_cache)
    if (e.ptr == ptr && e.pins > 0) {
      --e.pins;
      return;
    }
}

// test hook (dctadj_dense_cache_state): entries held / entries pinned now
static void dense_cache_state(int32_t* entries, int32_t* pinned) {
  std::lock_guard<std::mutex> lk(g_dense_mu);
  int np = 0;
  for (const auto& e : g_dense_cache) np += e.pins > 0;
  if (entries) *entries = static_cast<int32_t>(g_dense_cache.size());
  if (pinned) *pinned = np;
}

struct Launch {
  const KernelEntry* k = nullptr;
  LaunchArgs a;
  std::vector<unsigned char> row_coef, col_coef;
  void* dense_row = nullptr;  // pinned cache entries (released on reset / destruction)
  void* dense_col = nullptr;
  Launch() = default;
  Launch(const Launch&) = delete;
  Launch& operator=(const Launch&) = delete;
  ~Launch() { reset(); }
  void reset() {
    release_dense(dense_row);
    release_dense(dense_col);
    k = nullptr;
    a = LaunchArgs();
    row_coef.clear();
    col_coef.clear();
    dense_row = dense_col = nullptr;
  }
};

static int prepare(Launch& L, const AxisPlan& row, const AxisPlan* col, int dtype, int h, int w,
                   bool col_first, int in_mode, int out_mode, cudaStream_t st) {
  const int cc = col ? col->code : op_code(ST_NONE);
  L.k = find_kernel(dtype, h, w, row.code, cc, col_first ? 1 : 0, in_mode, out_mode);
  if (!L.k) return ST_ERR_UNSUPPORTED;
  L.row_coef = plan_coef(row, dtype);
  if (col) L.col_coef = plan_coef(*col, dtype);
  int rc = upload_dense(row, dtype, st, &L.dense_row);
  if (rc) return rc;
  if (col) {
    rc = upload_dense(*col, dtype, st, &L.dense_col);
    if (rc) return rc;
  }
  L.a.row_coef = L.row_coef.data();
  L.a.col_coef = col ? L.col_coef.data() : nullptr;
  L.a.dense_row = L.dense_row;
  L.a.dense_col = L.dense_col;
  L.a.stream = st;
  return ST_OK;
}

// the launch is enqueued: unpin its dense matrices (they stay cached)
static int finish(Launch& L, cudaStream_t st) {
  (void)st;
  L.reset();
  return ST_OK;
}

static int check_dtype(int dtype) {
  if (dtype != DT_F32 && dtype != DT_F64)
    return fail(ST_ERR_VALUE, "dtype must be DCTADJ_F32 or DCTADJ_F64, got %d", dtype);
  return ST_OK;
}

// ------------------------------------------------------------- 1-D batches
// TMA coordinates are 32-bit: a LINEAR launch covers at most this many rows;
// bigger batches run as several launches over consecutive sub-ranges
// (DCTADJ_MAX_ROWS lowers the limit, for tests)
static int64_t max_launch_rows() {
  static const int64_t v = [] {
    const char* s = std::getenv("DCTADJ_MAX_ROWS");
    const long long r = s ? std::atoll(s) : 0;
    return r > 0 ? static_cast<int64_t>(r) : (int64_t(1) << 30);
  }();
  return v;
}

// L.k->fn over `units` units of `unit_rows` rows / `unit_bytes` bytes each
static int launch_linear_chunked(Launch& L, const void* x, void* y, int64_t units,
                                 int64_t unit_rows, size_t unit_bytes) {
  const int64_t per = std::max<int64_t>(1, max_launch_rows() / unit_rows);
  for (int64_t u0 = 0; u0 < units; u0 += per) {
    const int64_t nu = std::min(per, units - u0);
    L.a.in = static_cast<const char*>(x) + static_cast<size_t>(u0) * unit_bytes;
    L.a.out = static_cast<char*>(y) + static_cast<size_t>(u0) * unit_bytes;
    L.a.rows = nu * unit_rows;
    if (int rc = L.k->fn(L.a)) return rc;
  }
  return ST_OK;
}

static int run_1d(const AxisPlan& plan, const void* x, void* y, int64_t nvec, int dtype,
                  cudaStream_t st) {
  if (nvec < 0) return fail(ST_ERR_SHAPE, "negative batch size %lld", (long long)nvec);
  if (nvec == 0) return ST_OK;
  if (!x || !y) return fail(ST_ERR_VALUE, "NULL data pointer");
  Launch L;
  int rc = prepare(L, plan, nullptr, dtype, 32, plan.n, false, MODE_LINEAR, MODE_LINEAR, st);
  if (rc == ST_ERR_UNSUPPORTED)
    return fail(rc, "no 1-D kernel for op 0x%x at n=%d dtype=%d", plan.code, plan.n, dtype);
  if (rc) return rc;
  rc = launch_linear_chunked(L, x, y, nvec, 1, static_cast<size_t>(plan.n) * dt_size(dtype));
  int rc2 = finish(L, st);
  return rc ? rc : rc2;
}

static int run_axis_1d(const dctadj_axis* ax, bool inverse, const void* x, void* y, int64_t nvec,
                       int dtype, cudaStream_t st) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  AxisPlan p;
  rc = plan_axis(ax, inverse, false, &p);
  if (rc) return rc;
  if (!find_kernel(dtype, 32, p.n, p.code, op_code(ST_NONE), 0, 0, 0)) {
    rc = plan_axis(ax, inverse, true, &p);
    if (rc) return rc;
  }
  return run_1d(p, x, y, nvec, dtype, st);
}

static int primitive(int stage, const void* x, void* y, int64_t nvec, int n, int dtype,
                     cudaStream_t st) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (n > 64) return fail(ST_ERR_VALUE, "size %d exceeds compiled kernel limit 64", n);
  if (!fast_size(n))
    return fail(ST_ERR_DIMENSION, "fast transforms support sizes (4, 8, 16, 32, 64), got %d", n);
  AxisPlan p;
  p.n = n;
  p.code = op_code(stage);
  p.gain_sq = n;
  return run_1d(p, x, y, nvec, dtype, st);
}

// ------------------------------------------------------------- dense on tensor cores
// DCTADJ_DENSE_TC=0 keeps the dense comparison path on the CUDA-core kernel (read
// per call: the Table-1 harness times both; getenv is a few ns beside a launch)
static bool dense_tc_enabled() {
  const char* s = std::getenv("DCTADJ_DENSE_TC");
  return !(s && s[0] == '0');
}

// one zeroed [next, done] counter pair per (device, stream): launches on one stream
// are ordered, and the last CTA of each launch re-zeroes it
static int stream_sched_counter(cudaStream_t st, unsigned long long** out) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, cudaStream_t>, unsigned long long*>> tab;
  int device = 0;
  DA_CUDA(cudaGetDevice(&device));
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : tab)
    if (e.first.first == device && e.first.second == st) {
      *out = e.second;
      return ST_OK;
    }
  unsigned long long* p = nullptr;
  DA_CUDA(cudaMalloc(&p, 2 * sizeof(unsigned long long)));
  DA_CUDA(cudaMemset(p, 0, 2 * sizeof(unsigned long long)));
  tab.push_back({{device, st}, p});
  *out = p;
  return ST_OK;
}

// ------------------------------------------------ cross-launch overlap (PDL)
// Every tile / ring / round-trip grid triggers its dependents at entry, so the
// next grid of the stream is scheduled while this one drains.  Normally the next
// grid then waits (griddepcontrol.wait) before touching memory.  When its byte
// ranges overlap none of the launches that may still be running on the stream
// -- every launch since the last one that waited at entry -- it may skip that
// wait (Geom::early) and wait at exit instead: its loads and passes fill the
// previous grid's tail, yet it never completes before it.  Ranges are per
// (device, stream); any other PDL-triggering launch poisons the record.  Other
// stream work (copies, events, kernels launched without the PDL attribute) is
// ordered normally by CUDA, which only makes the record conservative.
// DCTADJ_PDL_EARLY=0 disables the overlap.
namespace {
struct PdlLaunch {
  ByteRange in, out1, out2;
};
struct PdlStream {
  int device;
  cudaStream_t stream;
  bool poison;
  std::vector<PdlLaunch> live;  // since (and including) the last entry-waiting launch
};
std::mutex g_pdl_mu;
std::vector<PdlStream> g_pdl;
constexpr size_t kPdlMaxLive = 32;

bool pdl_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("DCTADJ_PDL_EARLY");
    return !(e && e[0] == '0');
  }();
  return v;
}
bool overlaps(ByteRange a, ByteRange b) {
  if (!a.p || !b.p || a.n == 0 || b.n == 0) return false;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a.p), b0 = reinterpret_cast<uintptr_t>(b.p);
  return a0 < b0 + b.n && b0 < a0 + a.n;
}
PdlStream& pdl_stream(cudaStream_t st) {
  int device = 0;
  cudaGetDevice(&device);
  for (auto& e : g_pdl)
    if (e.device == device && e.stream == st) return e;
  g_pdl.push_back({device, st, true, {}});  // unknown history: the first launch waits
  return g_pdl.back();
}
}  // namespace

bool pdl_early(cudaStream_t st, ByteRange in, ByteRange out1, ByteRange out2) {
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  PdlStream& r = pdl_stream(st);
  bool ok = pdl_enabled() && !r.poison && r.live.size() < kPdlMaxLive;
  for (size_t i = 0; ok && i < r.live.size(); ++i) {
    const PdlLaunch& p = r.live[i];
    // read-after-write, write-after-read, write-after-write
    if (overlaps(in, p.out1) || overlaps(in, p.out2) || overlaps(out1, p.in) ||
        overlaps(out1, p.out1) || overlaps(out1, p.out2) || overlaps(out2, p.in) ||
        overlaps(out2, p.out1) || overlaps(out2, p.out2))
      ok = false;
  }
  if (!ok) r.live.clear();
  r.poison = false;
  r.live.push_back({in, out1, out2});
  return ok;
}

void pdl_poison(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  PdlStream& r = pdl_stream(st);
  r.poison = true;
  r.live.clear();
}

// fused config-5 launch: the adjusted transform's output, packed coefficients
// (already in fp32) and the per-frame error accumulator
struct FusedArgs {
  void* adj_out;
  const void* row_coef;
  const void* col_coef;
  double* err;
};

// MMA-issuer poll back-off of the fused config-5 kernel (measured, tools/prof_fused.py)
constexpr int kFusedSpinNs = 0;
template <int IN_MODE, int OUT_MODE, int FRC = 0, int FCC = 0>
static int launch_dense_tc(const LaunchArgs& a, int64_t nblocks, int tiles_y, int tiles_x,
                           const FusedArgs* fz = nullptr) {
  constexpr int S = 8;  // ring of 8 x 16 KB + 4 group tiles x 16 KB: 208 KB, one CTA/SM
  Geom g{};
  g.nblocks = nblocks;
  g.ntiles = (nblocks + 3) / 4;
  g.tiles_y = tiles_y;
  g.tiles_x = tiles_x;
  LaunchArgs la = a;
  la.rows = nblocks * 32;
  CUtensorMap in_map, out_map;
  auto map_for = [&](CUtensorMap* m, const void* base, int mode) {
    if (mode == MODE_FRAME4) {  // {col in block, block column, frame row, frame}
      uint64_t dims[4] = {32, static_cast<uint64_t>(tiles_x), static_cast<uint64_t>(a.frame_h),
                          static_cast<uint64_t>(a.frames)};
      uint64_t strides[3] = {128, static_cast<uint64_t>(a.frame_w) * 4,
                             static_cast<uint64_t>(a.frame_w) * a.frame_h * 4};
      uint32_t box[4] = {32, 4, 32, 1};
      return encode_tensor_map(m, DT_F32, 4, dims, strides, box, 128, const_cast<void*>(base));
    }
    return mode == MODE_FRAME ? make_map<float, 32, 32, 4, MODE_FRAME>(m, base, la)
                              : make_map<float, 32, 32, 4, MODE_LINEAR>(m, base, la);
  };
  int rc = map_for(&in_map, a.in, IN_MODE);
  if (!rc) rc = map_for(&out_map, a.out, OUT_MODE);
  if (rc) return rc;
  CUtensorMap adj_map = in_map;  // unused unless fused
  KParams<float, 32, 32, FRC, FCC> kp;
  std::memset(&kp, 0, sizeof(kp));
  DenseTcParams prm{static_cast<const float*>(a.dense_row), static_cast<const float*>(a.dense_col),
                    nullptr, nullptr, nullptr, a.frame_h};
  if constexpr (FRC != 0) {
    if (!fz) return fail(ST_ERR_VALUE, "fused launch without its arguments");
    if ((rc = make_map<float, 32, 32, 4, MODE_LINEAR_IL>(&adj_map, fz->adj_out, la))) return rc;
    // the exact output is staged as an interleaved tile too (dense_tc.cuh, fused)
    if ((rc = make_map<float, 32, 32, 4, MODE_LINEAR_IL>(&out_map, a.out, la))) return rc;
    using RowOp = AxisOp<float, 32, FRC>;
    using ColOp = AxisOp<float, 32, FCC>;
    if (RowOp::NCOEF > 0) std::memcpy(kp.row.c, fz->row_coef, sizeof(float) * RowOp::NCOEF);
    if (ColOp::NCOEF > 0) std::memcpy(kp.col.c, fz->col_coef, sizeof(float) * ColOp::NCOEF);
    prm.err = fz->err;
  }
  int rc_s = stream_sched_counter(a.stream, &prm.sched);
  if (rc_s) return rc_s;
  // MMA-issuer back-off between polls (DCTADJ_TC_SPIN_NS overrides the default:
  // spin for the dense kernel, back off for the issue-bound fused one)
  static const char* spin_env = std::getenv("DCTADJ_TC_SPIN_NS");
  prm.spin_ns = spin_env ? std::atoi(spin_env) : (FRC != 0 ? kFusedSpinNs : 0);
  // diagnostics: DCTADJ_TC_TRACE=<file> dumps CTA 0's per-tile event clocks
  static const char* trace_file = std::getenv("DCTADJ_TC_TRACE");
  const size_t trace_bytes =
      sizeof(unsigned long long) * (kTcTraceTiles * kTcTraceEv + 2 * kTcTraceCtas);
  if (trace_file) {
    DA_CUDA(cudaMalloc(&prm.trace, trace_bytes));
    DA_CUDA(cudaMemsetAsync(prm.trace, 0, trace_bytes, a.stream));
  }
  constexpr int NG = kDenseTcGroups;
  constexpr int NTHR = (4 * NG + 3) * 32;
  auto kern = dense_tc_kernel<S, IN_MODE, OUT_MODE, FRC, FCC, NG>;
  const size_t smem = 1024 + S * 16384 + NG * 16384 + 16384 + (2 * S + 4 * NG) * 8 + (S + NG) * 8 +
                      NG * 16 * 8 + 16;
  static std::atomic<int> setup[kMaxDevices];  // per instantiation and device
  if (!kernel_blocks_per_sm(kern, NTHR, smem, setup, "dense_tc_kernel")) return ST_ERR_CUDA;
  const int bps = 1;  // the kernel allocates all 512 TMEM columns
  const int64_t cap = static_cast<int64_t>(num_sms_cached()) * bps;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(g.ntiles, cap)));
  cfg.blockDim = dim3(NTHR);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  pdl_poison(a.stream);
  DA_CUDA(cudaLaunchKernelEx(&cfg, kern, in_map, out_map, g, prm, adj_map, kp));
  if (trace_file) {
    std::vector<unsigned long long> h(kTcTraceTiles * kTcTraceEv + 2 * kTcTraceCtas);
    DA_CUDA(cudaMemcpyAsync(h.data(), prm.trace, trace_bytes, cudaMemcpyDeviceToHost, a.stream));
    DA_CUDA(cudaStreamSynchronize(a.stream));
    DA_CUDA(cudaFree(prm.trace));
    if (FILE* f = std::fopen(trace_file, "w")) {
      for (int k = 0; k < kTcTraceTiles; ++k) {
        for (int e = 0; e < kTcTraceEv; ++e) std::fprintf(f, "%llu ", h[k * kTcTraceEv + e]);
        std::fprintf(f, "\n");
      }
      // per-CTA start / end globaltimer (ns), 8 per line
      for (int c = 0; c < kTcTraceCtas; ++c) {
        for (int e = 0; e < 8; ++e)
          std::fprintf(f, "%llu ", e < 2 ? h[kTcTraceTiles * kTcTraceEv + 2 * c + e] : 0ull);
        std::fprintf(f, "\n");
      }
      std::fclose(f);
    }
  }
  return ST_OK;
}

#ifdef DCTADJ_TUNING
// config 5's fused step with role-specific register budgets (frames_exact.cuh)
template <int FRC, int FCC>
static int launch_frames_exact(const LaunchArgs& a, int64_t nblocks, int tiles_y, int tiles_x,
                               const FusedArgs& fz) {
  constexpr int S = 5;  // 5 x 16 KB ring + 2 x 2 exact 16 KB tiles + 8 adjusted 8 KB half-tiles: 224 KB
  Geom g{};
  g.nblocks = nblocks;
  g.ntiles = (nblocks + 3) / 4;
  g.tiles_y = tiles_y;
  g.tiles_x = tiles_x;
  if (g.ntiles == 0) return ST_OK;
  LaunchArgs la = a;
  la.rows = nblocks * 32;
  CUtensorMap in_map, out_map, adj_map;
  {  // frames: {col in block, block column, frame row, frame}, one box = 4 blocks
    uint64_t dims[4] = {32, static_cast<uint64_t>(tiles_x), static_cast<uint64_t>(a.frame_h),
                        static_cast<uint64_t>(a.frames)};
    uint64_t strides[3] = {128, static_cast<uint64_t>(a.frame_w) * 4,
                           static_cast<uint64_t>(a.frame_w) * a.frame_h * 4};
    uint32_t box[4] = {32, 4, 32, 1};
    int rc = encode_tensor_map(&in_map, DT_F32, 4, dims, strides, box, 128, const_cast<void*>(a.in));
    if (rc) return rc;
  }
  int rc = make_map<float, 32, 32, 4, MODE_LINEAR>(&out_map, a.out, la);
  if (!rc) rc = make_map<float, 32, 32, 2, MODE_LINEAR>(&adj_map, fz.adj_out, la);  // half-tiles
  if (rc) return rc;
  KParams<float, 32, 32, FRC, FCC> kp;
  std::memset(&kp, 0, sizeof(kp));
  using RowOp = AxisOp<float, 32, FRC>;
  using ColOp = AxisOp<float, 32, FCC>;
  if (RowOp::NCOEF > 0) std::memcpy(kp.row.c, fz.row_coef, sizeof(float) * RowOp::NCOEF);
  if (ColOp::NCOEF > 0) std::memcpy(kp.col.c, fz.col_coef, sizeof(float) * ColOp::NCOEF);
  DenseTcParams prm{static_cast<const float*>(a.dense_row), static_cast<const float*>(a.dense_col),
                    nullptr, nullptr, fz.err, a.frame_h, 0};
  if ((rc = stream_sched_counter(a.stream, &prm.sched))) return rc;
  auto kern = frames_exact_kernel<S, FRC, FCC>;
  constexpr size_t smem = frames_exact_smem<S>();
  static std::atomic<int> setup[kMaxDevices];
  if (!kernel_blocks_per_sm(kern, kFxThreads, smem, setup, "frames_exact_kernel")) return ST_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(g.ntiles, num_sms_cached())));
  cfg.blockDim = dim3(kFxThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  pdl_poison(a.stream);
  DA_CUDA(cudaLaunchKernelEx(&cfg, kern, in_map, out_map, g, prm, adj_map, kp));
  return ST_OK;
}
#endif  // DCTADJ_TUNING

// 64x64 fp32 dense on the tensor cores (dense_tc64.cuh), LINEAR blocks
static int launch_dense_tc64(const LaunchArgs& a, int64_t nblocks) {
  constexpr int S = 3;  // 3 x 32 KB ring + 2 x 32 KB staging + 64 KB matrices: 224 KB
  constexpr int NG = kTc64Groups;
  Geom g{};
  g.nblocks = nblocks;
  g.ntiles = (nblocks + 1) / 2;
  LaunchArgs la = a;
  la.rows = nblocks * 64;
  CUtensorMap in_map, out_map;
  int rc = make_map<float, 64, 64, 2, MODE_LINEAR>(&in_map, a.in, la);
  if (!rc) rc = make_map<float, 64, 64, 2, MODE_LINEAR>(&out_map, a.out, la);
  if (rc) return rc;
  DenseTcParams prm{static_cast<const float*>(a.dense_row), static_cast<const float*>(a.dense_col),
                    nullptr, nullptr, nullptr, 0};
  if ((rc = stream_sched_counter(a.stream, &prm.sched))) return rc;
  auto kern = dense_tc64_kernel<S>;
  const size_t smem = 1024 + S * 32768 + NG * 32768 + 65536 + (2 * S + 4 * NG) * 8 + (S + 1) * 8 + 16;
  static std::atomic<int> setup[kMaxDevices];  // per instantiation and device
  if (!kernel_blocks_per_sm(kern, kTc64Threads, smem, setup, "dense_tc64_kernel")) return ST_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(g.ntiles, num_sms_cached())));
  cfg.blockDim = dim3(kTc64Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  pdl_poison(a.stream);
  DA_CUDA(cudaLaunchKernelEx(&cfg, kern, in_map, out_map, g, prm));
  return ST_OK;
}

// ------------------------------------------------------------- 2-D / frames
static int run_2d(const dctadj_axis* h, const dctadj_axis* v, const void* x, void* y,
                  int64_t nblk, int dtype, bool inverse, int in_mode, int out_mode,
                  int32_t frames, int32_t fh, int32_t fw, cudaStream_t st) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  AxisPlan ph, pv;
  rc = plan_axis(h, inverse, false, &ph);
  if (rc) return rc;
  rc = plan_axis(v, inverse, false, &pv);
  if (rc) return rc;
  if (nblk < 0) return fail(ST_ERR_SHAPE, "negative block count %lld", (long long)nblk);
  if (nblk == 0) return ST_OK;
  if (!x || !y) return fail(ST_ERR_VALUE, "NULL data pointer");
  const int H = pv.n, W = ph.n;
  Launch L;
  if (dtype == DT_F32 && H == 64 && W == 64 && ph.code == op_code(ST_DENSE) &&
      pv.code == op_code(ST_DENSE) && dense_tc_enabled() && in_mode == MODE_LINEAR &&
      out_mode == MODE_LINEAR) {
    // 64x64 dense on the tensor cores (dense_tc64.cuh)
    if ((rc = upload_dense(ph, dtype, st, &L.dense_row)) || (rc = upload_dense(pv, dtype, st, &L.dense_col)))
      return rc;
    LaunchArgs a;
    a.dense_row = L.dense_row;
    a.dense_col = L.dense_col;
    a.stream = st;
    const int64_t per = std::max<int64_t>(2, max_launch_rows() / 64 / 2 * 2);  // whole super-tiles
    for (int64_t b0 = 0; b0 < nblk && !rc; b0 += per) {
      a.in = static_cast<const char*>(x) + static_cast<size_t>(b0) * 16384;
      a.out = static_cast<char*>(y) + static_cast<size_t>(b0) * 16384;
      rc = launch_dense_tc64(a, std::min(per, nblk - b0));
    }
    int rc2 = finish(L, st);
    return rc ? rc : rc2;
  }
  if (dtype == DT_F32 && H == 32 && W == 32 && ph.code == op_code(ST_DENSE) &&
      pv.code == op_code(ST_DENSE) && dense_tc_enabled() && in_mode != MODE_GATHER) {
    // the dense comparison path on the tensor cores (3xTF32 tcgen05, dense_tc.cuh)
    if ((rc = upload_dense(ph, dtype, st, &L.dense_row)) || (rc = upload_dense(pv, dtype, st, &L.dense_col)))
      return rc;
    LaunchArgs a;
    a.in = x;
    a.out = y;
    a.frames = frames;
    a.frame_h = fh;
    a.frame_w = fw;
    a.dense_row = L.dense_row;
    a.dense_col = L.dense_col;
    a.stream = st;
    const int ty = (fh + H - 1) / H, tx = fw / W;
    const bool f4 = tx % 4 == 0;  // super-tiles never straddle a block row
    if (in_mode == MODE_LINEAR && out_mode == MODE_LINEAR) {
      const int64_t per = std::max<int64_t>(4, max_launch_rows() / 32 / 4 * 4);  // whole super-tiles
      for (int64_t b0 = 0; b0 < nblk && !rc; b0 += per) {
        a.in = static_cast<const char*>(x) + static_cast<size_t>(b0) * 4096;
        a.out = static_cast<char*>(y) + static_cast<size_t>(b0) * 4096;
        rc = launch_dense_tc<MODE_LINEAR, MODE_LINEAR>(a, std::min(per, nblk - b0), 0, 0);
      }
    }
    else if (in_mode == MODE_FRAME)
      rc = f4 ? launch_dense_tc<MODE_FRAME4, MODE_LINEAR>(a, nblk, ty, tx)
              : launch_dense_tc<MODE_FRAME, MODE_LINEAR>(a, nblk, ty, tx);
    else
      rc = f4 ? launch_dense_tc<MODE_LINEAR, MODE_FRAME4>(a, nblk, ty, tx)
              : launch_dense_tc<MODE_LINEAR, MODE_FRAME>(a, nblk, ty, tx);
    int rc2 = finish(L, st);
    return rc ? rc : rc2;
  }
  if (in_mode == MODE_FRAME || out_mode == MODE_FRAME) {
    // frames: the interleaved one-box-per-super-tile kernel when the frame width
    // holds whole super-tiles (it declines otherwise), else the per-block boxes
    const int il_in = in_mode == MODE_FRAME ? MODE_FRAME_IL : MODE_LINEAR_IL;
    const int il_out = out_mode == MODE_FRAME ? MODE_FRAME_IL : MODE_LINEAR_IL;
    if (prepare(L, ph, &pv, dtype, H, W, inverse, il_in, il_out, st) == ST_OK) {
      L.a.in = x;
      L.a.out = y;
      L.a.rows = nblk * H;
      L.a.frames = frames;
      L.a.frame_h = fh;
      L.a.frame_w = fw;
      rc = L.k->fn(L.a);
      if (rc != ST_ERR_UNSUPPORTED) {
        int rc2 = finish(L, st);
        return rc ? rc : rc2;
      }
    }
    L.reset();
  }
  rc = prepare(L, ph, &pv, dtype, H, W, inverse, in_mode, out_mode, st);
  if (rc == ST_ERR_UNSUPPORTED) {
    // dense composite of both axes: one fused kernel per shape is always built
    rc = plan_axis(h, inverse, true, &ph);
    if (!rc) rc = plan_axis(v, inverse, true, &pv);
    if (rc) return rc;
    L.reset();
    rc = prepare(L, ph, &pv, dtype, H, W, inverse, in_mode, out_mode, st);
    if (rc == ST_ERR_UNSUPPORTED)
      return fail(rc, "no 2-D kernel for %dx%d blocks, dtype %d (mode %d->%d)", H, W, dtype,
                  in_mode, out_mode);
  }
  if (rc) return rc;
  L.a.frames = frames;
  L.a.frame_h = fh;
  L.a.frame_w = fw;
  if (in_mode == MODE_LINEAR && out_mode == MODE_LINEAR) {
    rc = launch_linear_chunked(L, x, y, nblk, H, static_cast<size_t>(H) * W * dt_size(dtype));
  } else {
    L.a.in = x;
    L.a.out = y;
    L.a.rows = nblk * H;
    rc = L.k->fn(L.a);
  }
  int rc2 = finish(L, st);
  return rc ? rc : rc2;
}

// ------------------------------------------------------------- round trip
// y = forward(x), xr = inverse(y) as ONE fused kernel (roundtrip.cuh) when one
// is built for these ops, else the two tile kernels back to back (identical
// results).  xr may alias x; y may not alias xr.  DCTADJ_RT_VARIANT=k picks a
// tuning variant, DCTADJ_RT_UNFUSED=1 forces the two-kernel path.
static int rt_variant() {
  static int v = [] {
    const char* s = std::getenv("DCTADJ_RT_VARIANT");
    return s ? std::atoi(s) : 0;
  }();
  return v;
}
static bool rt_unfused() {
  static bool v = [] {
    const char* s = std::getenv("DCTADJ_RT_UNFUSED");
    return s && s[0] == '1';
  }();
  return v;
}

static int run_roundtrip(const dctadj_axis* h, const dctadj_axis* v, const void* x, void* y,
                         void* xr, int64_t nblk, int dtype, cudaStream_t st) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  AxisPlan fh, fv, ih, iv;
  if ((rc = plan_axis(h, false, false, &fh)) || (rc = plan_axis(v, false, false, &fv)) ||
      (rc = plan_axis(h, true, false, &ih)) || (rc = plan_axis(v, true, false, &iv)))
    return rc;
  if (nblk < 0) return fail(ST_ERR_SHAPE, "negative block count %lld", (long long)nblk);
  if (nblk == 0) return ST_OK;
  if (!x || !y || !xr) return fail(ST_ERR_VALUE, "NULL data pointer");
  if (y == xr) return fail(ST_ERR_VALUE, "coefficients and reconstruction must not alias");
  const int H = fv.n, W = fh.n;
  const RtEntry* e = rt_unfused() ? nullptr
                                  : find_roundtrip(dtype, H, W, fh.code, fv.code, ih.code, iv.code,
                                                   MODE_LINEAR, rt_variant());
  if (trace_on())
    std::fprintf(stderr, "[dctadj] roundtrip dtype=%d %dx%d ops 0x%x/0x%x/0x%x/0x%x: %s\n", dtype, H,
                 W, fh.code, fv.code, ih.code, iv.code, e ? "fused" : "two kernels");
  if (!e) {
    rc = run_2d(h, v, x, y, nblk, dtype, false, MODE_LINEAR, MODE_LINEAR, 0, 0, 0, st);
    if (!rc) rc = run_2d(h, v, y, xr, nblk, dtype, true, MODE_LINEAR, MODE_LINEAR, 0, 0, 0, st);
    return rc;
  }
  const std::vector<unsigned char> c0 = plan_coef(fh, dtype), c1 = plan_coef(fv, dtype),
                                   c2 = plan_coef(ih, dtype), c3 = plan_coef(iv, dtype);
  RtArgs a;
  a.coef[0] = c0.data();
  a.coef[1] = c1.data();
  a.coef[2] = c2.data();
  a.coef[3] = c3.data();
  a.stream = st;
  const size_t bb = static_cast<size_t>(H) * W * dt_size(dtype);
  const int64_t per = std::max<int64_t>(1, max_launch_rows() / H);  // 32-bit TMA row range
  for (int64_t b0 = 0; b0 < nblk && !rc; b0 += per) {
    const int64_t nb = std::min(per, nblk - b0);
    a.in = static_cast<const char*>(x) + static_cast<size_t>(b0) * bb;
    a.y = static_cast<char*>(y) + static_cast<size_t>(b0) * bb;
    a.xr = static_cast<char*>(xr) + static_cast<size_t>(b0) * bb;
    a.rows = nb * H;
    rc = e->fn(a);
  }
  return rc;
}

// Host-buffer pipeline: chunks of blocks cycle through NSTREAM streams, each
// with its own device in/out buffers: H2D(c) overlaps kernel(c-1) and D2H(c-2)
// (PCIe is full duplex).  Streams and staging buffers persist per device
// (one pipeline at a time per device; concurrent host calls serialise).
struct HostPipe {
  static constexpr int NSTREAM = 8;  // capacity; host_streams() are used
  std::mutex mu;
  bool ready = false;
  cudaStream_t st[NSTREAM] = {};
  void* din[NSTREAM] = {};
  void* dout[NSTREAM] = {};
  size_t cap = 0;
};

static HostPipe& host_pipe(int device) {
  static HostPipe pipes[64];
  return pipes[(device >= 0 && device < 64) ? device : 0];
}

// streams in the host pipeline (DCTADJ_HOST_STREAMS, 2..8; default 4)
static int host_streams() {
  static const int v = [] {
    const char* s = std::getenv("DCTADJ_HOST_STREAMS");
    const int n = s ? std::atoi(s) : 4;
    return n < 2 ? 2 : n > 8 ? 8 : n;
  }();
  return v;
}

static size_t host_chunk_bytes() {
  static size_t v = [] {
    const char* s = std::getenv("DCTADJ_HOST_CHUNK_MB");
    const long mb = s ? std::atol(s) : 16;
    return static_cast<size_t>(mb > 0 ? mb : 16) << 20;
  }();
  return v;
}

// xrh != NULL (round trip, config 2): each chunk also runs the inverse on the
// device-resident coefficients and copies the reconstruction back, so the
// coefficients cross PCIe once (D2H) instead of three times.
// Blocks per pipeline chunk: full `chunk`s, with a ramp of 1/8, 1/4, 1/2 chunks
// at both ends of big batches so the first copy in and the last copies out
// (which nothing overlaps) are short.  DCTADJ_HOST_RAMP=0 turns the ramp off.
static std::vector<int64_t> host_chunk_schedule(int64_t nblk, int64_t chunk) {
  static const bool ramp = [] {
    const char* s = std::getenv("DCTADJ_HOST_RAMP");
    return !(s && s[0] == '0');
  }();
  std::vector<int64_t> head, tail, out;
  if (ramp && chunk >= 8 && nblk >= 4 * chunk) {
    head = {chunk / 8, chunk / 4, chunk / 2};
    tail = {chunk / 2, chunk / 4, chunk / 8};
  }
  int64_t mid = nblk;
  for (int64_t v : head) mid -= v;
  for (int64_t v : tail) mid -= v;
  out = head;
  for (int64_t b = 0; b < mid; b += chunk) out.push_back(std::min(chunk, mid - b));
  out.insert(out.end(), tail.begin(), tail.end());
  return out;
}

static int run_2d_host(const dctadj_axis* h, const dctadj_axis* v, const void* xh, void* yh,
                       int64_t nblk, int dtype, bool inverse, int device, void* xrh = nullptr) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if ((rc = validate_axis(h)) != ST_OK || (rc = validate_axis(v)) != ST_OK) return rc;
  if (nblk < 0) return fail(ST_ERR_SHAPE, "negative block count %lld", (long long)nblk);
  if (nblk == 0) return ST_OK;
  if (!xh || !yh) return fail(ST_ERR_VALUE, "NULL data pointer");
  DA_CUDA(cudaSetDevice(device));
  HostPipe& hp = host_pipe(device);
  std::lock_guard<std::mutex> lock(hp.mu);
  const size_t blk_bytes = static_cast<size_t>(h->n) * v->n * dt_size(dtype);
  const int64_t chunk = std::max<int64_t>(1, static_cast<int64_t>(host_chunk_bytes() / blk_bytes));
  const std::vector<int64_t> pieces = host_chunk_schedule(nblk, chunk);
  const int64_t nchunks = static_cast<int64_t>(pieces.size());
  const size_t need = static_cast<size_t>(chunk) * blk_bytes;
  if (!hp.ready) {
    for (int i = 0; i < HostPipe::NSTREAM; ++i)
      DA_CUDA(cudaStreamCreateWithFlags(&hp.st[i], cudaStreamNonBlocking));
    hp.ready = true;
  }
  if (hp.cap < need) {
    for (int i = 0; i < HostPipe::NSTREAM; ++i) {
      DA_CUDA(cudaStreamSynchronize(hp.st[i]));
      if (hp.din[i]) cudaFree(hp.din[i]);
      if (hp.dout[i]) cudaFree(hp.dout[i]);
      hp.din[i] = hp.dout[i] = nullptr;
    }
    hp.cap = 0;
    for (int i = 0; i < host_streams(); ++i) {
      DA_CUDA(cudaMalloc(&hp.din[i], need));
      DA_CUDA(cudaMalloc(&hp.dout[i], need));
    }
    hp.cap = need;
  }
  int status = ST_OK;
  int64_t b0 = 0;
  for (int64_t c = 0; c < nchunks && !status; b0 += pieces[c], ++c) {
    const int k = static_cast<int>(c % host_streams());
    const int64_t nb = pieces[c];
    const size_t off = static_cast<size_t>(b0) * blk_bytes, bytes = static_cast<size_t>(nb) * blk_bytes;
    if (cudaMemcpyAsync(hp.din[k], static_cast<const char*>(xh) + off, bytes,
                        cudaMemcpyHostToDevice, hp.st[k]) != cudaSuccess) {
      status = fail(ST_ERR_CUDA, "H2D copy: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    status = xrh ? run_roundtrip(h, v, hp.din[k], hp.dout[k], hp.din[k], nb, dtype, hp.st[k])
                 : run_2d(h, v, hp.din[k], hp.dout[k], nb, dtype, inverse, MODE_LINEAR,
                          MODE_LINEAR, 0, 0, 0, hp.st[k]);
    if (status) break;
    if (cudaMemcpyAsync(static_cast<char*>(yh) + off, hp.dout[k], bytes, cudaMemcpyDeviceToHost,
                        hp.st[k]) != cudaSuccess) {
      status = fail(ST_ERR_CUDA, "D2H copy: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    if (xrh) {  // reconstruction of the chunk: written over its consumed input
      if (cudaMemcpyAsync(static_cast<char*>(xrh) + off, hp.din[k], bytes, cudaMemcpyDeviceToHost,
                          hp.st[k]) != cudaSuccess)
        status = fail(ST_ERR_CUDA, "D2H copy: %s", cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int i = 0; i < HostPipe::NSTREAM; ++i) {
    cudaError_t e = cudaStreamSynchronize(hp.st[i]);
    if (e != cudaSuccess && !status) status = fail(ST_ERR_CUDA, "pipeline: %s", cudaGetErrorString(e));
  }
  return status;
}

static int run_frames(const dctadj_axis* h, const dctadj_axis* v, const void* in, void* out,
                      int32_t nframes, int32_t height, int32_t width, int dtype, bool inverse,
                      cudaStream_t st) {
  if (!h || !v) return fail(ST_ERR_VALUE, "axis descriptor is NULL");
  if (nframes < 0 || height < 0 || width < 0)
    return fail(ST_ERR_SHAPE, "negative frame geometry %d x %d x %d", nframes, height, width);
  if (nframes == 0 || height == 0 || width == 0) return ST_OK;
  if (width % h->n != 0)
    return fail(ST_ERR_SHAPE, "frame width %d is not a multiple of the block width %d", width,
                h->n);
  const int64_t nblk = static_cast<int64_t>(nframes) * ((height + v->n - 1) / v->n) * (width / h->n);
  return run_2d(h, v, in, out, nblk, dtype, inverse, inverse ? MODE_LINEAR : MODE_FRAME,
                inverse ? MODE_FRAME : MODE_LINEAR, nframes, height, width, st);
}

// ------------------------------------------------------------- frames: adjusted + exact
// Per-frame approximation error of adjusted vs exact coefficient blocks (the
// unfused path).  One warp walks a contiguous run of blocks; lane sums are
// flushed (warp-reduced, fp64 atomics) when the frame changes.
template <typename T>
__global__ void frame_err_kernel(const T* __restrict__ ya, const T* __restrict__ ye, double* err,
                                 int64_t nblk, int64_t per_frame, int tiles_x, int full_tile_rows,
                                 int64_t blocks_per_warp) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t b0 = warp * blocks_per_warp;
  const int64_t b1 = b0 + blocks_per_warp < nblk ? b0 + blocks_per_warp : nblk;
  double acc[4] = {0, 0, 0, 0};
  int cur = -1;
  auto flush = [&]() {
    for (int i = 0; i < 4; ++i) {
      double a = acc[i];
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0 && cur >= 0) atomicAdd(err + 4 * cur + i, a);
      acc[i] = 0;
    }
  };
  for (int64_t blk = b0; blk < b1; ++blk) {
    const int f = static_cast<int>(blk / per_frame);
    const int ty = static_cast<int>((blk - f * per_frame) / tiles_x);
    if (f != cur) {
      flush();
      cur = f;
    }
    double d2 = 0, e2 = 0;
    for (int i = lane; i < 1024; i += 32) {
      const double e = static_cast<double>(ye[blk * 1024 + i]);
      const double d = static_cast<double>(ya[blk * 1024 + i]) - e;
      d2 += d * d;
      e2 += e * e;
    }
    acc[0] += d2;
    acc[1] += e2;
    if (ty < full_tile_rows) {
      acc[2] += d2;
      acc[3] += e2;
    }
  }
  flush();
}

static int run_frames_exact(const dctadj_axis* h, const dctadj_axis* v, const dctadj_axis* eh,
                            const dctadj_axis* ev, const void* frames, void* coefs, void* exact,
                            double* err, int32_t nframes, int32_t height, int32_t width,
                            int32_t dtype, cudaStream_t st) {
  if (!h || !v || !eh || !ev) return fail(ST_ERR_VALUE, "axis descriptor is NULL");
  if (eh->n != h->n || ev->n != v->n)
    return fail(ST_ERR_SHAPE, "exact transforms (%d x %d) do not match the adjusted ones (%d x %d)",
                ev->n, eh->n, v->n, h->n);
  if (nframes < 0 || height < 0 || width < 0)
    return fail(ST_ERR_SHAPE, "negative frame geometry %d x %d x %d", nframes, height, width);
  if (err && nframes > 0) DA_CUDA(cudaMemsetAsync(err, 0, sizeof(double) * 4 * nframes, st));
  if (nframes == 0 || height == 0 || width == 0) return ST_OK;
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if ((rc = validate_axis(h)) || (rc = validate_axis(v)) || (rc = validate_axis(eh)) ||
      (rc = validate_axis(ev)))
    return rc;
  if (width % h->n != 0)
    return fail(ST_ERR_SHAPE, "frame width %d is not a multiple of the block width %d", width,
                h->n);
  const int ty = (height + v->n - 1) / v->n, tx = width / h->n;
  const int64_t nblk = static_cast<int64_t>(nframes) * ty * tx;
  if (!frames || !coefs || !exact) return fail(ST_ERR_VALUE, "NULL data pointer");

  // fused: one read of the frames feeds both transforms and the error sums
  // (dense_tc.cuh, FUSED).  Without err the two separate launches are faster
  // (each sits at the HBM roofline; the fused kernel is issue-bound).
  AxisPlan ph, pv, peh, pev;
  if (err && dtype == DT_F32 && h->n == 32 && v->n == 32 && tx % 4 == 0 && dense_tc_enabled() &&
      !plan_axis(h, false, false, &ph) && !plan_axis(v, false, false, &pv) &&
      !plan_axis(eh, false, true, &peh) && !plan_axis(ev, false, true, &pev) &&
      peh.code == op_code(ST_DENSE) && pev.code == op_code(ST_DENSE) && ph.code == pv.code) {
    constexpr int kSub8 = op_code(ST_DCT2, ST_SUB, 8), kGiv6 = op_code(ST_GIVENS2, ST_DST3, 6);
    if (ph.code == kSub8 || ph.code == kGiv6) {
      Launch L;
      if ((rc = upload_dense(peh, dtype, st, &L.dense_row)) ||
          (rc = upload_dense(pev, dtype, st, &L.dense_col)))
        return rc;
      std::vector<unsigned char> rcf = plan_coef(ph, DT_F32), ccf = plan_coef(pv, DT_F32);
      LaunchArgs a;
      a.in = frames;
      a.out = exact;
      a.frames = nframes;
      a.frame_h = height;
      a.frame_w = width;
      a.dense_row = L.dense_row;
      a.dense_col = L.dense_col;
      a.stream = st;
      FusedArgs fz{coefs, rcf.data(), ccf.data(), err};
      // the single-role fused kernel (dense_tc.cuh FUSED); the warp-specialised
      // variant (frames_exact.cuh, measured slower) only in DCTADJ_TUNING builds
#ifdef DCTADJ_TUNING
      static const bool ws = [] {
        const char* e = std::getenv("DCTADJ_FX_WS");
        return e && e[0] == '1';
      }();
      if (ws)
        rc = ph.code == kSub8 ? launch_frames_exact<kSub8, kSub8>(a, nblk, ty, tx, fz)
                              : launch_frames_exact<kGiv6, kGiv6>(a, nblk, ty, tx, fz);
      else
#endif
        rc = ph.code == kSub8
                 ? launch_dense_tc<MODE_FRAME4, MODE_LINEAR, kSub8, kSub8>(a, nblk, ty, tx, &fz)
                 : launch_dense_tc<MODE_FRAME4, MODE_LINEAR, kGiv6, kGiv6>(a, nblk, ty, tx, &fz);
      if (trace_on()) std::fprintf(stderr, "[dctadj] frames_exact: fused (rc %d)\n", rc);
      return rc;
    }
  }
  // the error sums are defined on 32x32 tiles (frame_err_kernel): refuse before any work
  if (err && (h->n != 32 || v->n != 32))
    return fail(ST_ERR_UNSUPPORTED,
                "per-frame error sums need 32x32 blocks, got %d x %d (pass err = NULL)", v->n,
                h->n);
  // unfused: two frame launches + the error reduction
  if ((rc = run_frames(h, v, frames, coefs, nframes, height, width, dtype, false, st))) return rc;
  if ((rc = run_frames(eh, ev, frames, exact, nframes, height, width, dtype, false, st))) return rc;
  if (err) {
    const int64_t per_warp = 64, warps = (nblk + per_warp - 1) / per_warp;
    const int grid = static_cast<int>((warps * 32 + 255) / 256);
    const int full = height / 32;
    if (dtype == DT_F32)
      frame_err_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(coefs),
                                                     static_cast<const float*>(exact), err, nblk,
                                                     static_cast<int64_t>(ty) * tx, tx, full, per_warp);
    else
      frame_err_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(coefs),
                                                      static_cast<const double*>(exact), err, nblk,
                                                      static_cast<int64_t>(ty) * tx, tx, full, per_warp);
    DA_CUDA(cudaGetLastError());
  }
  if (trace_on()) std::fprintf(stderr, "[dctadj] frames_exact: unfused\n");
  return ST_OK;
}

// ------------------------------------------------------------- encoder evaluation
template <typename T, int H, int W, int P, int NG, int S>
static int launch_enc5(const void* x, void* const* outs, int64_t nblk, const double* cv,
                       const double* ch, cudaStream_t st) {
  using L = TileLayout<T, H, W, P>;
  Geom g{};
  g.ntiles = (nblk * H + L::PH - 1) / L::PH;
  g.nblocks = g.ntiles * P;
  LaunchArgs a;
  a.rows = nblk * H;
  CUtensorMap in_map, om[5];
  int rc = make_map<T, H, W, P, MODE_LINEAR>(&in_map, x, a);
  for (int i = 0; i < 5 && !rc; ++i) rc = make_map<T, H, W, P, MODE_LINEAR>(&om[i], outs[i], a);
  if (rc) return rc;
  Enc5Params<T> prm;
  for (int i = 0; i < 64; ++i) {
    prm.cv[i] = static_cast<T>(cv[i]);
    prm.ch[i] = static_cast<T>(ch[i]);
  }
  auto kern = enc5_kernel<T, H, W, P, NG, S>;
  const size_t smem = 1024 + static_cast<size_t>(NG) * (S + 4) * L::STAGEB + NG * S * 8;
  static std::atomic<int> setup[kMaxDevices];  // per instantiation and device
  const int bps = kernel_blocks_per_sm(kern, NG * 32, smem, setup, "enc5_kernel");
  if (!bps) return ST_ERR_CUDA;
  const int64_t want = (g.ntiles + NG - 1) / NG;
  const int64_t cap = static_cast<int64_t>(num_sms_cached()) * bps;
  kern<<<static_cast<int>(std::min(want, cap)), NG * 32, smem, st>>>(in_map, om[0], om[1], om[2],
                                                                    om[3], om[4], g, prm);
  DA_CUDA(cudaGetLastError());
  return ST_OK;
}

using Enc5Fn = int (*)(const void*, void* const*, int64_t, const double*, const double*,
                       cudaStream_t);
struct Enc5Entry {
  int dtype, h, w;
  Enc5Fn fn;
};
static const Enc5Entry kEnc5[] = {
    {0, 16, 16, &launch_enc5<float, 16, 16, 2, 4, 2>},
    {0, 16, 32, &launch_enc5<float, 16, 32, 2, 4, 2>},
    {0, 32, 16, &launch_enc5<float, 32, 16, 2, 4, 2>},
    {0, 32, 32, &launch_enc5<float, 32, 32, 1, 4, 2>},
    {0, 32, 64, &launch_enc5<float, 32, 64, 1, 2, 2>},
    {0, 64, 32, &launch_enc5<float, 64, 32, 1, 2, 2>},
    {0, 64, 64, &launch_enc5<float, 64, 64, 1, 1, 2>},
    {1, 16, 16, &launch_enc5<double, 16, 16, 2, 2, 2>},
    {1, 32, 32, &launch_enc5<double, 32, 32, 1, 2, 2>},
    {1, 32, 64, &launch_enc5<double, 32, 64, 1, 1, 2>},
    {1, 64, 32, &launch_enc5<double, 64, 32, 1, 1, 2>},
    {1, 64, 64, &launch_enc5<double, 64, 64, 1, 1, 2>},
};

static int check_enc_axis(const dctadj_axis* a, const char* name) {
  int rc = validate_axis(a);
  if (rc) return rc;
  if (a->adj != DCTADJ_ADJ_SUBBLOCK)
    return fail(ST_ERR_CONFIG, "%s adjustment must be a sub-block design", name);
  if (a->side != DCTADJ_SIDE_POST || a->base != DCTADJ_BASE_DCT2)
    return fail(ST_ERR_CONFIG, "%s adjustment must be post-side dct2 -> dst7", name);
  return ST_OK;
}

// C8 = S C7 S of a post sub-block axis (reference design.py:677-715)
static void chessboard(const dctadj_axis* a, std::vector<double>& m8) {
  const int n = a->n;
  m8.assign(a->mat, a->mat + static_cast<size_t>(n) * n);
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < n; ++j)
      if ((r + j) & 1) m8[r * n + j] = -m8[r * n + j];
}

static int run_enc5(const dctadj_axis* h, const dctadj_axis* v, const void* x, void* const* outs,
                    int64_t nblk, int dtype, cudaStream_t st) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if ((rc = check_enc_axis(h, "horizontal")) || (rc = check_enc_axis(v, "vertical"))) return rc;
  if (nblk < 0) return fail(ST_ERR_SHAPE, "negative block count");
  if (nblk == 0) return ST_OK;
  if (!x || !outs) return fail(ST_ERR_VALUE, "NULL data pointer");
  for (int i = 0; i < 5; ++i)
    if (!outs[i]) return fail(ST_ERR_VALUE, "NULL output plane %d", i);
  if (h->order == 8 && v->order == 8) {
    for (const Enc5Entry& e : kEnc5)
      if (e.dtype == dtype && e.h == v->n && e.w == h->n) {
        double cv[64], ch[64];
        for (int r = 0; r < 8; ++r)
          for (int j = 0; j < 8; ++j) {
            cv[r * 8 + j] = v->mat[r * v->n + j];
            ch[r * 8 + j] = h->mat[r * h->n + j];
          }
        return e.fn(x, outs, nblk, cv, ch, st);
      }
  }
  // general sub-block orders / shapes: five fused 2-D transforms
  std::vector<double> h8, v8;
  chessboard(h, h8);
  chessboard(v, v8);
  dctadj_axis h7 = *h, v7 = *v, hd = *h, vd = *v, h8a = *h, v8a = *v;
  hd.adj = vd.adj = DCTADJ_ADJ_NONE;
  h8a.mat = h8.data();
  v8a.mat = v8.data();
  const dctadj_axis* hs[5] = {&hd, &h7, &h8a, &h7, &h8a};
  const dctadj_axis* vs[5] = {&vd, &v7, &v7, &v8a, &v8a};
  for (int i = 0; i < 5; ++i)
    if ((rc = run_2d(hs[i], vs[i], x, outs[i], nblk, dtype, false, MODE_LINEAR, MODE_LINEAR, 0, 0,
                     0, st)))
      return rc;
  return ST_OK;
}

// ------------------------------------------------------------- mixed batches
}  // namespace dctadj

struct dctadj_mixed {
  struct Class {
    int32_t h_index, v_index;
    int64_t count;
    int64_t* offsets;  // device, into `all`
  };
  std::vector<Class> classes;
  std::vector<int32_t> sizes;
  int64_t total_elements = 0;
  int64_t nblk = 0;
  int64_t* all = nullptr;  // device
  int device = 0;
  // class kernels run concurrently on NSTREAM streams forked from the caller's
  // stream (their persistent grids fill each other's tails)
  static constexpr int NSTREAM = 4;
  cudaStream_t aux[NSTREAM] = {};
  cudaEvent_t fork = nullptr;
  cudaEvent_t join[NSTREAM] = {};
};

namespace dctadj {

static int run_mixed(const dctadj_mixed* plan, const dctadj_axis* table, const void* x, void* y,
                     int dtype, bool inverse, cudaStream_t st) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (!plan || !table) return fail(ST_ERR_VALUE, "NULL plan or axis table");
  for (size_t k = 0; k < plan->sizes.size(); ++k) {
    if ((rc = validate_axis(&table[k])) != ST_OK) return rc;
    if (table[k].n != plan->sizes[k])
      return fail(ST_ERR_SHAPE, "axis table entry %zu has n=%d, plan built for %d", k,
                  table[k].n, plan->sizes[k]);
  }
  if (plan->nblk == 0) return ST_OK;
  if (!x || !y) return fail(ST_ERR_VALUE, "NULL data pointer");
  DA_CUDA(cudaEventRecord(plan->fork, st));
  for (int i = 0; i < dctadj_mixed::NSTREAM; ++i) DA_CUDA(cudaStreamWaitEvent(plan->aux[i], plan->fork, 0));
  int ci = 0;
  for (const auto& c : plan->classes) {
    cudaStream_t cs = plan->aux[ci++ % dctadj_mixed::NSTREAM];
    const dctadj_axis* h = &table[c.h_index];
    const dctadj_axis* v = &table[c.v_index];
    AxisPlan ph, pv;
    if ((rc = plan_axis(h, inverse, false, &ph)) || (rc = plan_axis(v, inverse, false, &pv))) return rc;
    Launch L;
    rc = prepare(L, ph, &pv, dtype, v->n, h->n, inverse, MODE_GATHER, MODE_GATHER, cs);
    if (rc == ST_ERR_UNSUPPORTED) {
      if ((rc = plan_axis(h, inverse, true, &ph)) || (rc = plan_axis(v, inverse, true, &pv))) return rc;
      L.reset();
      rc = prepare(L, ph, &pv, dtype, v->n, h->n, inverse, MODE_GATHER, MODE_GATHER, cs);
      if (rc == ST_ERR_UNSUPPORTED)
        return fail(rc, "no gather kernel for %dx%d blocks, dtype %d", v->n, h->n, dtype);
    }
    if (rc) return rc;
    L.a.in = x;
    L.a.out = y;
    L.a.rows = plan->total_elements / h->n;
    L.a.offsets = c.offsets;
    L.a.gather_blocks = c.count;
    rc = L.k->fn(L.a);
    int rc2 = finish(L, cs);
    if (rc || rc2) return rc ? rc : rc2;
  }
  for (int i = 0; i < dctadj_mixed::NSTREAM; ++i) {
    DA_CUDA(cudaEventRecord(plan->join[i], plan->aux[i]));
    DA_CUDA(cudaStreamWaitEvent(st, plan->join[i], 0));
  }
  return ST_OK;
}

struct MixedRtClass {
  const RtEntry* e = nullptr;
  AxisPlan fh, fv, ih, iv;
};
// the fused gather kernel of every class, or *fused = false when one is missing
static int plan_mixed_roundtrip(const dctadj_mixed* plan, const dctadj_axis* table, int dtype,
                                std::vector<MixedRtClass>& runs, bool* fused) {
  runs.assign(plan->classes.size(), MixedRtClass());
  *fused = !rt_unfused();
  for (size_t i = 0; i < plan->classes.size() && *fused; ++i) {
    const auto& c = plan->classes[i];
    const dctadj_axis* h = &table[c.h_index];
    const dctadj_axis* v = &table[c.v_index];
    MixedRtClass& r = runs[i];
    int rc;
    if ((rc = plan_axis(h, false, false, &r.fh)) || (rc = plan_axis(v, false, false, &r.fv)) ||
        (rc = plan_axis(h, true, false, &r.ih)) || (rc = plan_axis(v, true, false, &r.iv)))
      return rc;
    r.e = find_roundtrip(dtype, v->n, h->n, r.fh.code, r.fv.code, r.ih.code, r.iv.code,
                         MODE_GATHER, rt_variant());
    *fused = r.e != nullptr;
  }
  return ST_OK;
}

// Mixed batch round trip: y = forward(x), xr = inverse(y) per class as ONE
// fused gather kernel (roundtrip.cuh) when every class has one, else the
// forward and inverse mixed runs back to back (identical results).
static int run_mixed_roundtrip(const dctadj_mixed* plan, const dctadj_axis* table, const void* x,
                               void* y, void* xr, int dtype, cudaStream_t st) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (!plan || !table) return fail(ST_ERR_VALUE, "NULL plan or axis table");
  for (size_t k = 0; k < plan->sizes.size(); ++k) {
    if ((rc = validate_axis(&table[k])) != ST_OK) return rc;
    if (table[k].n != plan->sizes[k])
      return fail(ST_ERR_SHAPE, "axis table entry %zu has n=%d, plan built for %d", k,
                  table[k].n, plan->sizes[k]);
  }
  if (plan->nblk == 0) return ST_OK;
  if (!x || !y || !xr) return fail(ST_ERR_VALUE, "NULL data pointer");
  if (y == xr) return fail(ST_ERR_VALUE, "coefficients and reconstruction must not alias");
  std::vector<MixedRtClass> runs;
  bool fused = false;
  if ((rc = plan_mixed_roundtrip(plan, table, dtype, runs, &fused))) return rc;
  if (trace_on())
    std::fprintf(stderr, "[dctadj] mixed roundtrip: %s\n", fused ? "fused" : "two passes");
  if (!fused) {
    rc = run_mixed(plan, table, x, y, dtype, false, st);
    return rc ? rc : run_mixed(plan, table, y, xr, dtype, true, st);
  }
  DA_CUDA(cudaEventRecord(plan->fork, st));
  for (int i = 0; i < dctadj_mixed::NSTREAM; ++i) DA_CUDA(cudaStreamWaitEvent(plan->aux[i], plan->fork, 0));
  for (size_t i = 0; i < plan->classes.size(); ++i) {
    const auto& c = plan->classes[i];
    const MixedRtClass& r = runs[i];
    const std::vector<unsigned char> c0 = plan_coef(r.fh, dtype), c1 = plan_coef(r.fv, dtype),
                                     c2 = plan_coef(r.ih, dtype), c3 = plan_coef(r.iv, dtype);
    RtArgs a;
    a.in = x;
    a.y = y;
    a.xr = xr;
    a.rows = plan->total_elements / r.fh.n;
    a.coef[0] = c0.data();
    a.coef[1] = c1.data();
    a.coef[2] = c2.data();
    a.coef[3] = c3.data();
    a.offsets = c.offsets;
    a.gather_blocks = c.count;
    a.stream = plan->aux[i % dctadj_mixed::NSTREAM];
    if ((rc = r.e->fn(a))) return rc;
  }
  for (int i = 0; i < dctadj_mixed::NSTREAM; ++i) {
    DA_CUDA(cudaEventRecord(plan->join[i], plan->aux[i]));
    DA_CUDA(cudaStreamWaitEvent(st, plan->join[i], 0));
  }
  return ST_OK;
}

// generic rectangular dense product (rows != n), the one path off the tile kernel
template <typename T>
__global__ void dense_rect_kernel(const T* __restrict__ m, int rows, const T* __restrict__ x,
                                  T* __restrict__ y, int64_t nvec, int n) {
  const int64_t total = nvec * rows;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / rows;
    const int r = static_cast<int>(e - i * rows);
    T acc = m[r * n] * x[i * n];
    for (int j = 1; j < n; ++j) acc = fma(m[r * n + j], x[i * n + j], acc);
    y[e] = acc;
  }
}

}  // namespace dctadj

using namespace dctadj;

static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

int dctadj_dct2(const void* x, void* y, int64_t nvec, int32_t n, int32_t dtype, void* stream) {
  return primitive(ST_DCT2, x, y, nvec, n, dtype, S(stream));
}
int dctadj_idct2(const void* x, void* y, int64_t nvec, int32_t n, int32_t dtype, void* stream) {
  return primitive(ST_IDCT2, x, y, nvec, n, dtype, S(stream));
}
int dctadj_dst3(const void* x, void* y, int64_t nvec, int32_t n, int32_t dtype, void* stream) {
  return primitive(ST_DST3, x, y, nvec, n, dtype, S(stream));
}
int dctadj_idst3(const void* x, void* y, int64_t nvec, int32_t n, int32_t dtype, void* stream) {
  return primitive(ST_IDST3, x, y, nvec, n, dtype, S(stream));
}

int dctadj_band(const double* a, int32_t taps, const void* x, void* y, int64_t nvec, int32_t n,
                int32_t dtype, void* stream) {
  dctadj_axis ax{n, DCTADJ_BASE_DCT2, DCTADJ_ADJ_BAND, DCTADJ_SIDE_PRE, taps, 0, a, nullptr, 0, 0};
  int rc = check_dtype(dtype);
  if (rc) return rc;
  rc = validate_axis(&ax);
  if (rc) return rc;
  AxisPlan p;
  p.n = n;
  if (taps == 4 || taps == 6) {
    p.code = op_code(ST_BAND, ST_NONE, taps);
    pack_band(&ax, false, taps, p.coef);
    if (find_kernel(dtype, 32, n, p.code, 0, 0, 0, 0)) return run_1d(p, x, y, nvec, dtype, S(stream));
  }
  // any other width: the band-masked matrix as a dense product
  p.code = op_code(ST_DENSE);
  p.coef.clear();
  p.dense.assign(static_cast<size_t>(n) * n, 0.0);
  for (int r = 0; r < n; ++r)
    for (int j = 0; j < n; ++j)
      if (std::abs(r - j) < taps) p.dense[r * n + j] = a[r * n + j];
  return run_1d(p, x, y, nvec, dtype, S(stream));
}

int dctadj_subblock(const double* blk, int32_t b, const void* x, void* y, int64_t nvec,
                    int32_t n, int32_t dtype, void* stream) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (!fast_size(n))
    return fail(ST_ERR_DIMENSION, "fast transforms support sizes (4, 8, 16, 32, 64), got %d", n);
  if (b < 1 || b > n) return fail(ST_ERR_PATTERN, "sub-block order must be in 1..%d, got %d", n, b);
  if (!blk) return fail(ST_ERR_VALUE, "sub-block pointer is NULL");
  AxisPlan p;
  p.n = n;
  if (b == 8) {
    p.code = op_code(ST_SUB, ST_NONE, 8);
    p.coef.assign(blk, blk + 64);
    if (find_kernel(dtype, 32, n, p.code, 0, 0, 0, 0)) return run_1d(p, x, y, nvec, dtype, S(stream));
  }
  p.code = op_code(ST_DENSE);
  p.coef.clear();
  p.dense.assign(static_cast<size_t>(n) * n, 0.0);
  for (int r = 0; r < n; ++r) p.dense[r * n + r] = 1.0;
  for (int r = 0; r < b; ++r)
    for (int j = 0; j < b; ++j) p.dense[r * n + j] = blk[r * b + j];
  return run_1d(p, x, y, nvec, dtype, S(stream));
}

int dctadj_dense(const double* m, int32_t rows, const void* x, void* y, int64_t nvec, int32_t n,
                 int32_t dtype, void* stream) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (!m) return fail(ST_ERR_VALUE, "matrix pointer is NULL");
  if (rows < 1 || n < 1) return fail(ST_ERR_SHAPE, "bad dense shape %d x %d", rows, n);
  if (nvec < 0) return fail(ST_ERR_SHAPE, "negative batch size");
  if (nvec == 0) return ST_OK;
  if (rows == n && fast_size(n)) {
    AxisPlan p;
    p.n = n;
    p.code = op_code(ST_DENSE);
    p.dense.assign(m, m + static_cast<size_t>(n) * n);
    return run_1d(p, x, y, nvec, dtype, S(stream));
  }
  cudaStream_t st = S(stream);
  std::vector<double> md(m, m + static_cast<size_t>(rows) * n);
  AxisPlan p;
  p.dense = md;
  void* dm = nullptr;
  rc = upload_dense(p, dtype, st, &dm);
  if (rc) return rc;
  const int64_t total = nvec * rows;
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  if (dtype == DT_F32)
    dense_rect_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(dm), rows,
                                                    static_cast<const float*>(x),
                                                    static_cast<float*>(y), nvec, n);
  else
    dense_rect_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(dm), rows,
                                                     static_cast<const double*>(x),
                                                     static_cast<double*>(y), nvec, n);
  release_dense(dm);  // the launch is enqueued
  DA_CUDA(cudaGetLastError());
  return ST_OK;
}

int dctadj_forward_1d(const dctadj_axis* ax, const void* x, void* y, int64_t nvec, int32_t dtype,
                      void* stream) {
  return run_axis_1d(ax, false, x, y, nvec, dtype, S(stream));
}
int dctadj_inverse_1d(const dctadj_axis* ax, const void* y, void* x, int64_t nvec, int32_t dtype,
                      void* stream) {
  return run_axis_1d(ax, true, y, x, nvec, dtype, S(stream));
}

int dctadj_forward_2d(const dctadj_axis* h, const dctadj_axis* v, const void* x, void* y,
                      int64_t nblk, int32_t dtype, void* stream) {
  return run_2d(h, v, x, y, nblk, dtype, false, MODE_LINEAR, MODE_LINEAR, 0, 0, 0, S(stream));
}
int dctadj_inverse_2d(const dctadj_axis* h, const dctadj_axis* v, const void* y, void* x,
                      int64_t nblk, int32_t dtype, void* stream) {
  return run_2d(h, v, y, x, nblk, dtype, true, MODE_LINEAR, MODE_LINEAR, 0, 0, 0, S(stream));
}
int dctadj_roundtrip_fused(const dctadj_axis* h, const dctadj_axis* v, int32_t dtype) {
  AxisPlan fh, fv, ih, iv;
  if (check_dtype(dtype) || plan_axis(h, false, false, &fh) || plan_axis(v, false, false, &fv) ||
      plan_axis(h, true, false, &ih) || plan_axis(v, true, false, &iv))
    return 0;
  return !rt_unfused() &&
         find_roundtrip(dtype, fv.n, fh.n, fh.code, fv.code, ih.code, iv.code, MODE_LINEAR,
                        rt_variant()) != nullptr;
}
int dctadj_roundtrip_2d(const dctadj_axis* h, const dctadj_axis* v, const void* x, void* y,
                        void* xr, int64_t nblk, int32_t dtype, void* stream) {
  return run_roundtrip(h, v, x, y, xr, nblk, dtype, S(stream));
}

int dctadj_forward_2d_host(const dctadj_axis* h, const dctadj_axis* v, const void* x_host,
                           void* y_host, int64_t nblk, int32_t dtype, int32_t device) {
  return run_2d_host(h, v, x_host, y_host, nblk, dtype, false, device);
}
int dctadj_inverse_2d_host(const dctadj_axis* h, const dctadj_axis* v, const void* y_host,
                           void* x_host, int64_t nblk, int32_t dtype, int32_t device) {
  return run_2d_host(h, v, y_host, x_host, nblk, dtype, true, device);
}
int dctadj_roundtrip_2d_host(const dctadj_axis* h, const dctadj_axis* v, const void* x_host,
                             void* y_host, void* xr_host, int64_t nblk, int32_t dtype,
                             int32_t device) {
  if (!xr_host && nblk > 0) return fail(ST_ERR_VALUE, "NULL data pointer");
  return run_2d_host(h, v, x_host, y_host, nblk, dtype, false, device, xr_host);
}

int dctadj_forward_frames(const dctadj_axis* h, const dctadj_axis* v, const void* frames,
                          void* coefs, int32_t nframes, int32_t height, int32_t width,
                          int32_t dtype, void* stream) {
  return run_frames(h, v, frames, coefs, nframes, height, width, dtype, false, S(stream));
}
int dctadj_inverse_frames(const dctadj_axis* h, const dctadj_axis* v, const void* coefs,
                          void* frames, int32_t nframes, int32_t height, int32_t width,
                          int32_t dtype, void* stream) {
  return run_frames(h, v, coefs, frames, nframes, height, width, dtype, true, S(stream));
}
int dctadj_forward_frames_exact(const dctadj_axis* h, const dctadj_axis* v, const dctadj_axis* eh,
                                const dctadj_axis* ev, const void* frames, void* coefs,
                                void* exact, double* err, int32_t nframes, int32_t height,
                                int32_t width, int32_t dtype, void* stream) {
  return run_frames_exact(h, v, eh, ev, frames, coefs, exact, err, nframes, height, width, dtype,
                          S(stream));
}

int dctadj_copy_tiles(const void* x, void* y, int64_t nblk, int32_t h, int32_t w, int32_t dtype,
                      void* stream) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (nblk < 0) return fail(ST_ERR_SHAPE, "negative block count");
  if (nblk == 0) return ST_OK;
  AxisPlan ph, pv;
  ph.n = w;
  pv.n = h;
  ph.code = pv.code = op_code(ST_NONE);
  Launch L;
  rc = prepare(L, ph, &pv, dtype, h, w, false, MODE_LINEAR, MODE_LINEAR, S(stream));
  if (rc == ST_ERR_UNSUPPORTED) return fail(rc, "no copy kernel for %dx%d", h, w);
  if (rc) return rc;
  L.a.in = x;
  L.a.out = y;
  L.a.rows = nblk * h;
  return L.k->fn(L.a);
}

int dctadj_encoder_eval(const dctadj_axis* h, const dctadj_axis* v, const void* x,
                        void* const* planes, int64_t nblk, int32_t dtype, void* stream) {
  return run_enc5(h, v, x, planes, nblk, dtype, S(stream));
}

int dctadj_mixed_create(const int64_t* offsets, const int32_t* h_index, const int32_t* v_index,
                        int64_t nblk, const int32_t* sizes, int32_t ntable,
                        int64_t total_elements, dctadj_mixed** out) {
  if (!out) return fail(ST_ERR_VALUE, "NULL plan output");
  *out = nullptr;
  if (nblk < 0 || ntable < 1 || total_elements < 0)
    return fail(ST_ERR_SHAPE, "bad mixed batch geometry");
  if (nblk > 0 && (!offsets || !h_index || !v_index || !sizes))
    return fail(ST_ERR_VALUE, "NULL descriptor array");
  for (int k = 0; k < ntable; ++k)
    if (!fast_size(sizes[k]))
      return fail(ST_ERR_DIMENSION, "fast transforms support sizes (4, 8, 16, 32, 64), got %d",
                  sizes[k]);
  // bucket by (h, v) class: counting sort on the host, once
  std::vector<int64_t> count(static_cast<size_t>(ntable) * ntable, 0);
  for (int64_t i = 0; i < nblk; ++i) {
    const int hi = h_index[i], vi = v_index[i];
    if (hi < 0 || hi >= ntable || vi < 0 || vi >= ntable)
      return fail(ST_ERR_VALUE, "block %lld: axis index out of range", (long long)i);
    const int64_t w = sizes[hi], hgt = sizes[vi];
    if (offsets[i] < 0 || offsets[i] % w != 0 || offsets[i] + hgt * w > total_elements)
      return fail(ST_ERR_SHAPE, "block %lld: offset %lld does not fit a %lldx%lld block in %lld elements",
                  (long long)i, (long long)offsets[i], (long long)hgt, (long long)w,
                  (long long)total_elements);
    if (total_elements % w != 0)
      return fail(ST_ERR_SHAPE, "buffer of %lld elements is not a whole number of %lld-wide rows",
                  (long long)total_elements, (long long)w);
    ++count[hi * ntable + vi];
  }
  auto* plan = new dctadj_mixed();
  plan->sizes.assign(sizes, sizes + ntable);
  plan->total_elements = total_elements;
  plan->nblk = nblk;
  cudaGetDevice(&plan->device);
  std::vector<int64_t> start(count.size() + 1, 0);
  for (size_t c = 0; c < count.size(); ++c) start[c + 1] = start[c] + count[c];
  std::vector<int64_t> sorted(static_cast<size_t>(nblk));
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  for (int64_t i = 0; i < nblk; ++i) sorted[fill[h_index[i] * ntable + v_index[i]]++] = offsets[i];
  if (nblk > 0) {
    if (cudaMalloc(&plan->all, sizeof(int64_t) * nblk) != cudaSuccess ||
        cudaMemcpy(plan->all, sorted.data(), sizeof(int64_t) * nblk, cudaMemcpyHostToDevice) !=
            cudaSuccess) {
      cudaFree(plan->all);
      delete plan;
      return fail(ST_ERR_CUDA, "mixed plan upload: %s", cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int hi = 0; hi < ntable; ++hi)
    for (int vi = 0; vi < ntable; ++vi) {
      const size_t c = static_cast<size_t>(hi) * ntable + vi;
      if (count[c]) plan->classes.push_back({hi, vi, count[c], plan->all + start[c]});
    }
  // largest classes first (longest-processing-time order across the streams)
  std::stable_sort(plan->classes.begin(), plan->classes.end(),
                   [&](const dctadj_mixed::Class& a, const dctadj_mixed::Class& b) {
                     return a.count * plan->sizes[a.h_index] * plan->sizes[a.v_index] >
                            b.count * plan->sizes[b.h_index] * plan->sizes[b.v_index];
                   });
  bool ok = cudaEventCreateWithFlags(&plan->fork, cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; ok && i < dctadj_mixed::NSTREAM; ++i)
    ok = cudaStreamCreateWithFlags(&plan->aux[i], cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&plan->join[i], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    dctadj_mixed_destroy(plan);
    return fail(ST_ERR_CUDA, "mixed plan streams: %s", cudaGetErrorString(cudaGetLastError()));
  }
  *out = plan;
  return ST_OK;
}

int dctadj_mixed_forward(const dctadj_mixed* plan, const dctadj_axis* table, const void* x,
                         void* y, int32_t dtype, void* stream) {
  return run_mixed(plan, table, x, y, dtype, false, S(stream));
}
int dctadj_mixed_inverse(const dctadj_mixed* plan, const dctadj_axis* table, const void* y,
                         void* x, int32_t dtype, void* stream) {
  return run_mixed(plan, table, y, x, dtype, true, S(stream));
}
int dctadj_mixed_roundtrip(const dctadj_mixed* plan, const dctadj_axis* table, const void* x,
                           void* y, void* xr, int32_t dtype, void* stream) {
  return run_mixed_roundtrip(plan, table, x, y, xr, dtype, S(stream));
}
int dctadj_mixed_roundtrip_fused(const dctadj_mixed* plan, const dctadj_axis* table,
                                 int32_t dtype) {
  if (!plan || !table || check_dtype(dtype)) return 0;
  for (size_t k = 0; k < plan->sizes.size(); ++k)
    if (validate_axis(&table[k]) != ST_OK || table[k].n != plan->sizes[k]) return 0;
  std::vector<MixedRtClass> runs;
  bool fused = false;
  return plan_mixed_roundtrip(plan, table, dtype, runs, &fused) == ST_OK && fused;
}
int dctadj_mixed_destroy(dctadj_mixed* plan) {
  if (!plan) return ST_OK;
  for (int i = 0; i < dctadj_mixed::NSTREAM; ++i) {
    if (plan->aux[i]) {
      cudaStreamSynchronize(plan->aux[i]);
      cudaStreamDestroy(plan->aux[i]);
    }
    if (plan->join[i]) cudaEventDestroy(plan->join[i]);
  }
  if (plan->fork) cudaEventDestroy(plan->fork);
  if (plan->all) cudaFree(plan->all);
  delete plan;
  return ST_OK;
}

const char* dctadj_status_string(int32_t status) {
  switch (status) {
    case DCTADJ_OK: return "ok";
    case DCTADJ_ERR_DIMENSION: return "InvalidDimensionError";
    case DCTADJ_ERR_SHAPE: return "ShapeError";
    case DCTADJ_ERR_PATTERN: return "PatternError";
    case DCTADJ_ERR_CONFIG: return "ConfigurationError";
    case DCTADJ_ERR_KIND: return "KindMismatchError";
    case DCTADJ_ERR_CUDA: return "CudaError";
    case DCTADJ_ERR_UNSUPPORTED: return "Unsupported";
    case DCTADJ_ERR_VALUE: return "ValueError";
    default: return "unknown";
  }
}
const char* dctadj_last_error(void) { return g_err; }
int32_t dctadj_version(void) { return 1; }
int32_t dctadj_kernel_count(void) {
  int32_t n = 0;
  for (const KernelEntry& e : kRegistry) n += (e.variant == 0);
  return n;
}
int dctadj_dense_cache_state(int32_t* entries, int32_t* pinned) {
  dense_cache_state(entries, pinned);
  return ST_OK;
}
int dctadj_pdl_probe(void* stream, const void* in, uint64_t in_bytes, const void* out,
                     uint64_t out_bytes, int32_t poison) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (poison) {
    pdl_poison(st);
    return 0;
  }
  return pdl_early(st, {in, static_cast<size_t>(in_bytes)}, {out, static_cast<size_t>(out_bytes)})
             ? 1 : 0;
}
int32_t dctadj_tuning_build(void) {
#ifdef DCTADJ_TUNING
  return 1;
#else
  return 0;
#endif
}

}  // extern "C"

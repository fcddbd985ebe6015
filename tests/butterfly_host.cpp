// CPU harness for csrc/butterfly.cuh (test infrastructure): the device butterflies
// and the adjusted-axis stages compiled for the host through a small shim, so their
// arithmetic -- including the scaled / deferred-scale rotations and the host-side
// Givens packing that absorbs the deferred scales -- is unit-tested without a GPU.
// Built by tests/test_butterfly_host.py with g++ -std=c++17.
#include <cmath>
#include <cstring>
#include <vector>

#define __device__
#define __host__
#define __forceinline__ inline
#define __restrict__
struct float2 {
  float x, y;
};
static inline float2 make_float2(float x, float y) { return {x, y}; }
static inline float2 __fadd2_rn(float2 a, float2 b) { return {a.x + b.x, a.y + b.y}; }
static inline float2 __fmul2_rn(float2 a, float2 b) { return {a.x * b.x, a.y * b.y}; }
static inline float2 __ffma2_rn(float2 a, float2 b, float2 c) {
  return {std::fmaf(a.x, b.x, c.x), std::fmaf(a.y, b.y, c.y)};
}
using std::fma;
using std::fmaf;

#include "../paper_2505_23618_b200/csrc/givens_pack.h"

using namespace dctadj;

template <typename V> struct Lane;
template <> struct Lane<float> {
  static float in(double v) { return static_cast<float>(v); }
  static double out(float v) { return v; }
};
template <> struct Lane<double> {
  static double in(double v) { return v; }
  static double out(double v) { return v; }
};
template <> struct Lane<f2> {  // lane x carries the vector, lane y its negation (both checked)
  static f2 in(double v) { return {make_float2(static_cast<float>(v), static_cast<float>(-v))}; }
  static double out(f2 v) { return v.v.x == -v.v.y ? v.v.x : NAN; }
};

template <typename V, int N, int CODE>
static void run(const double* coef, const double* x, double* y) {
  using S = typename Scalar<V>::type;
  using Op = AxisOp<S, N, CODE>;
  typename Op::Coef cf;
  for (int i = 0; i < Op::NCOEF; ++i) cf.c[i] = static_cast<S>(coef[i]);
  V v[N];
  for (int i = 0; i < N; ++i) v[i] = Lane<V>::in(x[i]);
  apply_axis<V, N, CODE>(v, cf, nullptr);
  for (int i = 0; i < N; ++i) y[i] = Lane<V>::out(v[i]);
}

template <int N, int CODE>
static int run_v(int vtype, const double* coef, const double* x, double* y) {
  if (vtype == 0) run<float, N, CODE>(coef, x, y);
  else if (vtype == 1) run<double, N, CODE>(coef, x, y);
  else run<f2, N, CODE>(coef, x, y);
  return 0;
}

template <int N>
static int run_n(int s1, int s2, int k, int vtype, const double* coef, const double* x, double* y) {
#define CASE(A, B, K) \
  if (s1 == A && s2 == B && k == K) return run_v<N, op_code(A, B, K)>(vtype, coef, x, y);
  CASE(ST_DCT2, ST_NONE, 0)
  CASE(ST_IDCT2, ST_NONE, 0)
  CASE(ST_DST3, ST_NONE, 0)
  CASE(ST_IDST3, ST_NONE, 0)
  if constexpr (N >= 8) {
    CASE(ST_DCT2, ST_SUB, 8)
    CASE(ST_SUB, ST_IDCT2, 8)
  }
  if constexpr (N >= 16) {
    CASE(ST_GIVENS2, ST_DST3, 6)
    CASE(ST_IDST3, ST_GIVENS2, 6)
    CASE(ST_GIVENS2, ST_IDCT2, 6)
    CASE(ST_DCT2, ST_GIVENS2, 6)
    CASE(ST_GIVENS2, ST_DST3, 4)
    CASE(ST_IDST3, ST_GIVENS2, 4)
  }
#undef CASE
  return -1;
}

extern "C" {
// one vector through apply_axis<V, n, op_code(s1, s2, k)>; vtype 0 float, 1 double, 2 packed f2
int bf_apply(int n, int s1, int s2, int k, int vtype, const double* coef, const double* x,
             double* y) {
  switch (n) {
    case 4: return run_n<4>(s1, s2, k, vtype, coef, x, y);
    case 8: return run_n<8>(s1, s2, k, vtype, coef, x, y);
    case 16: return run_n<16>(s1, s2, k, vtype, coef, x, y);
    case 32: return run_n<32>(s1, s2, k, vtype, coef, x, y);
    case 64: return run_n<64>(s1, s2, k, vtype, coef, x, y);
    default: return -1;
  }
}
// abi.cu's packing rule for a band given as its Givens schedule; returns the count (0: refused)
int bf_pack_givens2(int n, int k, const double* givens, int inverse, double gain, int base_before,
                    double* out, int cap) {
  std::vector<double> c;
  if (!pack_givens2(n, k, givens, inverse != 0, gain, base_before, c)) return 0;
  if (static_cast<int>(c.size()) > cap) return -1;
  std::memcpy(out, c.data(), c.size() * sizeof(double));
  return static_cast<int>(c.size());
}
// the kernels' (type, size) choice of butterfly form (butterfly.cuh): which element types run
// the deferred-scale base in front of a Givens stage / the scaled inverse rotations
int bf_deferred_policy(int is_double, int n) { return deferred_policy(is_double != 0, n); }
int bf_idct_scaled_policy(int is_double, int n) { return idct_scaled_policy(is_double != 0, n); }
// abi.cu's rule for an 8 x 8 block behind the deferred DCT-2 (in place)
void bf_fold_sub(int n, int k, double* block) {
  std::vector<double> b(block, block + k * k);
  fold_sub_scales(n, k, b);
  std::memcpy(block, b.data(), b.size() * sizeof(double));
}
double bf_deferred_scale(int n, int s1, int j) {
  return s1 == ST_IDST3 ? deferred_scale_of<ST_IDST3>(n, j) : deferred_scale_of<ST_DCT2>(n, j);
}
// both inverse forms, whatever the policy picks: scaled != 0 -> idct2s, else idct2p (double)
int bf_idct2(int n, int scaled, const double* y, double* x) {
#define RUN(N)                                                      \
  if (n == N) {                                                     \
    double v[N], o[N];                                              \
    for (int i = 0; i < N; ++i) v[i] = y[i];                        \
    if (scaled) idct2s<double, N>(v, o); else idct2p<double, N>(v, o); \
    for (int i = 0; i < N; ++i) x[i] = o[i];                        \
    return 0;                                                       \
  }
  RUN(4) RUN(8) RUN(16) RUN(32) RUN(64)
#undef RUN
  return -1;
}
// the deferred forward DCT-2 alone: held outputs and their scales (n = 8..64)
int bf_dct2d(int n, int alt, const double* x, double* held, double* scale) {
#define RUN(N)                                                                 \
  if (n == N) {                                                                \
    double v[N], y[N];                                                         \
    for (int i = 0; i < N; ++i) v[i] = x[i];                                   \
    if (alt) dct2d<double, ScAlt, N>(v, y); else dct2d<double, ScUnit, N>(v, y); \
    for (int i = 0; i < N; ++i) {                                              \
      held[i] = y[i];                                                          \
      scale[i] = alt ? dct2d_out_scale<N, true>(i) : dct2d_out_scale<N, false>(i); \
    }                                                                          \
    return 0;                                                                  \
  }
  RUN(2) RUN(4) RUN(8) RUN(16) RUN(32) RUN(64)
#undef RUN
  return -1;
}
}

// butterfly.cuh -- register-resident fast DCT-2 / DCT-3 butterflies and the
// per-axis adjusted-transform stages (band, sub-block, dense).
//
// One thread owns one length-N vector as a register array; every index below
// is a compile-time constant after unrolling, so the arrays live in registers
// and the twiddles fold into FFMA immediates (fp32) or constant-bank operands
// (fp64).  The factorization is the reference's (same recursion, same
// per-output arithmetic order, FMA-contracted):
//   dct2  <- reference kernels/_fastcore.pyx:50-84   (even/odd split)
//   dct4  <- reference kernels/_fastcore.pyx:87-117  (pair rotations + half DCT-2/DST-2)
//   idct2 <- reference kernels/_fastcore.pyx:120-152
//   idct4 <- reference kernels/_fastcore.pyx:155-185
//   dst3  <- reference kernels/_fastcore.pyx:214-230 (reverse, idct2, negate odd)
//   idst3 <- reference kernels/_fastcore.pyx:233-250 (negate odd, dct2, reverse)
//   band  <- reference kernels/_fastcore.pyx:253-273 (ascending-j in-band sum)
//   sub   <- reference kernels/_fastcore.pyx:276-290 (leading BxB, tail untouched)
// Two forms of each butterfly live here: the plain ones (dct2u / dct4u, idct2p / idct4p:
// the reference's rotations as 2 multiplies + 2 FMAs) and the scaled ones (idct2s / idct4s:
// cosines absorbed by the parent's butterflies; dct2d / dct4d: compile-time deferred scales
// absorbed by the stage behind, or finalized with one multiply per output).  Which one a
// kernel gets is decided by (element type, size) alone -- idct_scaled_policy /
// deferred_policy -- so every kernel family computes a transform with the same arithmetic.
#pragma once
#include <cstdint>
#include <type_traits>

#include "twiddles.h"

namespace dctadj {

#define DA_DEV __device__ __forceinline__

// ---------------------------------------------------------------------------
// Value types.  V is the per-thread element: float, double, or f2 -- two fp32
// lanes (two adjacent columns, or two rows) processed by one packed
// FADD2/FMUL2/FFMA2 instruction (sm_100).  Scalars (twiddles, adjustment
// coefficients) are S = float/double and broadcast into both lanes (an
// immediate or a uniform-register operand of the packed instruction).
struct f2 {
  float2 v;
};
template <typename V> struct Scalar { using type = V; };
template <> struct Scalar<f2> { using type = float; };

DA_DEV float add(float a, float b) { return a + b; }
DA_DEV float sub(float a, float b) { return a - b; }
DA_DEV float neg(float a) { return -a; }
DA_DEV float mul(float a, float c) { return a * c; }
DA_DEV float fmac(float a, float c, float b) { return fmaf(a, c, b); }    // a*c + b
DA_DEV float fnmac(float a, float c, float b) { return fmaf(-a, c, b); }  // b - a*c
DA_DEV double add(double a, double b) { return a + b; }
DA_DEV double sub(double a, double b) { return a - b; }
DA_DEV double neg(double a) { return -a; }
DA_DEV double mul(double a, double c) { return a * c; }
DA_DEV double fmac(double a, double c, double b) { return fma(a, c, b); }
DA_DEV double fnmac(double a, double c, double b) { return fma(-a, c, b); }
DA_DEV f2 add(f2 a, f2 b) { return {__fadd2_rn(a.v, b.v)}; }
DA_DEV f2 sub(f2 a, f2 b) { return {__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))}; }
DA_DEV f2 neg(f2 a) { return {make_float2(-a.v.x, -a.v.y)}; }
DA_DEV f2 mul(f2 a, float c) { return {__fmul2_rn(a.v, make_float2(c, c))}; }
DA_DEV f2 fmac(f2 a, float c, f2 b) { return {__ffma2_rn(a.v, make_float2(c, c), b.v)}; }
DA_DEV f2 fnmac(f2 a, float c, f2 b) { return {__ffma2_rn(a.v, make_float2(-c, -c), b.v)}; }

// Unnormalized recursion.  The reference scales by 1/sqrt(2) at every level
// (u = (a+b)/sqrt2, v = (a-b)/sqrt2, and (c +- s)/sqrt2 in the DCT-4 output
// butterflies): ~125 of the 411 flops of a 32-point DCT-2.  Dropping those
// scalings makes every routine below return sqrt(N) x the orthonormal result,
// uniformly over its outputs (induction: dct2u_N = sqrt2 * {dct2u_N/2, dct4u_N/2}
// needs g(dct2u_M) == g(dct4u_M); the bases give g = 2 at M = 4, and dct4u only
// needs its two unscaled outputs y[0], y[M-1] multiplied by sqrt2).  The gain is
// removed once per launch (1/32 for a 32x32 block, exact in binary).
template <typename V, int N> DA_DEV void dct2u(const V (&x)[N], V (&y)[N]);
template <typename V, int M> DA_DEV void dct4u(const V (&x)[M], V (&y)[M]);
template <typename V, int N> DA_DEV void idct2u(const V (&y)[N], V (&x)[N]);

// DCT-2, gain sqrt(N): structure of reference _fastcore.pyx:50-84
template <typename V, int N>
DA_DEV void dct2u(const V (&x)[N], V (&y)[N]) {
  using S = typename Scalar<V>::type;
  if constexpr (N == 1) {
    y[0] = x[0];
  } else if constexpr (N == 2) {
    y[0] = add(x[0], x[1]);
    y[1] = sub(x[0], x[1]);
  } else if constexpr (N == 4) {
    constexpr S A = S(K_A4X2), B = S(K_B4X2);
    const V s03 = add(x[0], x[3]), d03 = sub(x[0], x[3]);
    const V s12 = add(x[1], x[2]), d12 = sub(x[1], x[2]);
    y[0] = add(s03, s12);
    y[2] = sub(s03, s12);
    y[1] = fmac(d03, A, mul(d12, B));
    y[3] = fnmac(d12, A, mul(d03, B));
  } else {
    constexpr int H = N / 2;
    V u[H], v[H], eu[H], ov[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      u[i] = add(x[i], x[N - 1 - i]);
      v[i] = sub(x[i], x[N - 1 - i]);
    }
    dct2u<V, H>(u, eu);
    dct4u<V, H>(v, ov);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      y[2 * i] = eu[i];
      y[2 * i + 1] = ov[i];
    }
  }
}

// DCT-4, gain sqrt(M): structure of reference _fastcore.pyx:87-117
template <typename V, int M>
DA_DEV void dct4u(const V (&x)[M], V (&y)[M]) {
  static_assert(M >= 4, "dct4u is only reached from dct2u with N >= 8");
  using S = typename Scalar<V>::type;
  constexpr int H = M / 2;
  constexpr int OFF = psi_off(M);
  constexpr S SQ2 = S(K_SQRT2);
  V p[H], sq[H], c[H], s2[H];
#pragma unroll
  for (int n = 0; n < H; ++n) {
    const V a = x[n], b = x[M - 1 - n];
    const S cp = S(psi_c(OFF + n)), sp = S(psi_s(OFF + n));
    p[n] = fmac(a, cp, mul(b, sp));
    // q = b cp - a sp; DST2(q) = reverse(DCT2(sign-alternated q))
    sq[n] = (n % 2 == 0) ? fnmac(a, sp, mul(b, cp)) : fnmac(b, cp, mul(a, sp));
  }
  dct2u<V, H>(p, c);
  dct2u<V, H>(sq, s2);
  y[0] = mul(c[0], SQ2);
#pragma unroll
  for (int r = 1; r < H; ++r) {
    y[2 * r] = add(c[r], s2[H - r]);
    y[2 * r - 1] = sub(c[r], s2[H - r]);
  }
  y[2 * H - 1] = mul(s2[0], -SQ2);
}

// ---------------------------------------------------------------------------
// Forward DCT-2 with DEFERRED scales (round 2; dct2d / dct4d).  In the forward
// direction the rotations open the DCT-4, so their cosines cannot be absorbed by
// a following add; instead every value carries a compile-time scale (held h,
// true value s * h): an add / subtract of two values with scales a, b becomes
// one FMA, h_a +- (b / a) h_b, with scale a; a rotation becomes two independent
// FMAs whose results carry c * a and c * b; the sqrt2 multiplies of the DCT-4
// end outputs disappear into their scales.  All ratios are constants, so a
// 32-point transform is 186 instructions instead of 242 -- but its outputs come
// out as y[k] = Dct2dOut<In, N>::at(k) * held[k].  Three consumers (apply_axis /
// run_stage below): the scaled-rotation band stage takes per-sample input scales
// for free (ST_GIVENS2: the host starts its scale tracking from them,
// givens_pack.h); the sub-block post-adjustment gets them folded into its
// block's columns by the host and finalizes only the untouched tail; a stage on
// its own finalizes every output (one multiply where the scale is not 1: 216).
// `In` types give the input scales: ScUnit, or ScAlt for the sign alternation
// of idst3 (a free negation).
struct ScUnit {
  static __host__ __device__ constexpr double at(int) { return 1.0; }
};
struct ScAlt {
  static __host__ __device__ constexpr double at(int i) { return i % 2 ? -1.0 : 1.0; }
};
template <class In, int M>
struct ScRotP {  // p = cp a + sp b = (cp a_s) (A + rho B)
  static __host__ __device__ constexpr double at(int n) { return psi_c(psi_off(M) + n) * In::at(n); }
};
template <class In, int M>
struct ScRotQ {  // (+-) q = (+-) (cp b - sp a) = (+-)(cp b_s) (B - rho A): DST-2 sign alternation in the scale
  static __host__ __device__ constexpr double at(int n) {
    return (n % 2 ? -1.0 : 1.0) * psi_c(psi_off(M) + n) * In::at(M - 1 - n);
  }
};
template <class In, int N> struct Dct2dOut;
template <class In, int M>
struct Dct4dOut {
  using C = Dct2dOut<ScRotP<In, M>, M / 2>;
  using Q = Dct2dOut<ScRotQ<In, M>, M / 2>;
  static __host__ __device__ constexpr double at(int k) {
    return k == 0 ? K_SQRT2 * C::at(0) : k == M - 1 ? -K_SQRT2 * Q::at(0) : C::at((k + 1) / 2);
  }
};
template <class In, int N>
struct Dct2dOut {
  static __host__ __device__ constexpr double at(int k) {
    if constexpr (N == 1 || N == 2) {
      return In::at(0);
    } else if constexpr (N == 4) {
      return k == 1 ? K_A4X2 * In::at(0) : k == 3 ? -K_A4X2 * In::at(1) : In::at(0);
    } else {
      return k % 2 == 0 ? Dct2dOut<In, N / 2>::at(k / 2) : Dct4dOut<In, N / 2>::at(k / 2);
    }
  }
};

template <int I, int E, class F>
DA_DEV void static_for(F&& f) {
  if constexpr (I < E) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, E>(f);
  }
}

// sum = a + r b, diff = a - r b for a compile-time ratio (plain add / subtract when |r| = 1)
#define DA_BFLY(a, b, r, sum, diff)        \
  if constexpr ((r) == S(1)) {             \
    sum = add(a, b);                       \
    diff = sub(a, b);                      \
  } else if constexpr ((r) == S(-1)) {     \
    sum = sub(a, b);                       \
    diff = add(a, b);                      \
  } else {                                 \
    sum = fmac(b, r, a);                   \
    diff = fnmac(b, r, a);                 \
  }

template <typename V, class In, int N> DA_DEV void dct2d(const V (&x)[N], V (&y)[N]);

template <typename V, class In, int M>
DA_DEV void dct4d(const V (&x)[M], V (&y)[M]) {
  static_assert(M >= 4, "dct4d is only reached from dct2d with N >= 8");
  using S = typename Scalar<V>::type;
  constexpr int H = M / 2;
  constexpr int OFF = psi_off(M);
  using PS = ScRotP<In, M>;
  using QS = ScRotQ<In, M>;
  V p[H], sq[H], c[H], s2[H];
  static_for<0, H>([&](auto ic) {
    constexpr int n = decltype(ic)::value;
    constexpr double t = psi_s(OFF + n) / psi_c(OFF + n), a = In::at(n), b = In::at(M - 1 - n);
    constexpr S rp = S(t * b / a), rq = S(t * a / b);
    p[n] = fmac(x[M - 1 - n], rp, x[n]);
    sq[n] = fnmac(x[n], rq, x[M - 1 - n]);
  });
  dct2d<V, PS, H>(p, c);
  dct2d<V, QS, H>(sq, s2);
  using CO = Dct2dOut<PS, H>;
  using QO = Dct2dOut<QS, H>;
  y[0] = c[0];
  static_for<1, H>([&](auto ic) {
    constexpr int r = decltype(ic)::value;
    constexpr S rho = S(QO::at(H - r) / CO::at(r));
    DA_BFLY(c[r], s2[H - r], rho, y[2 * r], y[2 * r - 1])
  });
  y[2 * H - 1] = s2[0];
}

template <typename V, class In, int N>
DA_DEV void dct2d(const V (&x)[N], V (&y)[N]) {
  using S = typename Scalar<V>::type;
  if constexpr (N == 1) {
    y[0] = x[0];
  } else if constexpr (N == 2) {
    constexpr S r = S(In::at(1) / In::at(0));
    DA_BFLY(x[0], x[1], r, y[0], y[1])
  } else if constexpr (N == 4) {
    constexpr double a0 = In::at(0), a1 = In::at(1), a2 = In::at(2), a3 = In::at(3);
    constexpr double BA = K_B4X2 / K_A4X2;
    constexpr S r03 = S(a3 / a0), r12 = S(a2 / a1), r10 = S(a1 / a0);
    V s03, d03, s12, d12;
    DA_BFLY(x[0], x[3], r03, s03, d03)  // scale a0
    DA_BFLY(x[1], x[2], r12, s12, d12)  // scale a1
    DA_BFLY(s03, s12, r10, y[0], y[2])  // a0
    y[1] = fmac(d12, S(BA * a1 / a0), d03);           // A a0 (d03 + (B a1 / A a0) d12)
    y[3] = fnmac(d03, S(BA * a0 / a1), d12);          // -A a1 (d12 - (B a0 / A a1) d03)
  } else {
    constexpr int H = N / 2;
    V u[H], v[H], eu[H], ov[H];
    static_for<0, H>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      constexpr S r = S(In::at(N - 1 - i) / In::at(i));
      DA_BFLY(x[i], x[N - 1 - i], r, u[i], v[i])
    });
    dct2d<V, In, H>(u, eu);
    dct4d<V, In, H>(v, ov);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      y[2 * i] = eu[i];
      y[2 * i + 1] = ov[i];
    }
  }
}

#undef DA_BFLY

// out[k] = scale_k * held[k] for k >= FROM (one multiply, none where the scale is 1);
// REV: out[j] = the value of held[N - 1 - j] (idst3's output reversal)
template <typename V, class In, int N, int FROM, bool REV>
DA_DEV void finalize_deferred(const V (&held)[N], V (&out)[N]) {
  using S = typename Scalar<V>::type;
  static_for<FROM, N>([&](auto ic) {
    constexpr int k = decltype(ic)::value;
    constexpr double sg = Dct2dOut<In, N>::at(k);
    constexpr int o = REV ? N - 1 - k : k;
    if constexpr (sg == 1.0)
      out[o] = held[k];
    else
      out[o] = mul(held[k], S(sg));
  });
}

// y[k] = dct2d_out_scale<N, ALT>(k) * held[k] after dct2d<V, ScUnit | ScAlt, N> (host: the
// initial scales of the Givens stage that follows)
template <int N, bool ALT>
__host__ __device__ constexpr double dct2d_out_scale(int k) {
  return ALT ? Dct2dOut<ScAlt, N>::at(k) : Dct2dOut<ScUnit, N>::at(k);
}

// Scaled rotations (round 2).  A DCT-4 pair rotation (c, s) = (cos psi, sin psi) is
// c * [[1, -t], [t, 1]] with t = tan psi < 1: two independent FMAs once the factor
// c is carried as a scale of both outputs.  In the inverse (DCT-3) direction the
// rotations are the LAST step of the inverse DCT-4 and its outputs only feed the parent's
// add / subtract butterflies, x = u +- v: with v = c v' those become FMAs, so the
// scale costs nothing (2 instructions per rotation instead of 4; 46 of the 242 of
// a 32-point transform).  idct4s returns v' and idct4_scale<M>(i) the factor of
// output i (negative where the reference's sign alternation lands).
template <int M>
__host__ __device__ constexpr double idct4_scale(int i) {
  const int n = i < M / 2 ? i : M - 1 - i;
  const double c = psi_c(psi_off(M) + n);
  return (i >= M / 2 && n % 2 == 1) ? -c : c;
}
template <typename V, int M> DA_DEV void idct4s(const V (&y)[M], V (&x)[M]);
template <typename V, int N> DA_DEV void idct2s(const V (&y)[N], V (&x)[N]);
template <typename V, int N> DA_DEV void idct2p(const V (&y)[N], V (&x)[N]);

// DCT-3 (inverse DCT-2), gain sqrt(N), scaled rotations: structure of reference _fastcore.pyx:120-152
template <typename V, int N>
DA_DEV void idct2s(const V (&y)[N], V (&x)[N]) {
  using S = typename Scalar<V>::type;
  if constexpr (N == 1) {
    x[0] = y[0];
  } else if constexpr (N == 2) {
    x[0] = add(y[0], y[1]);
    x[1] = sub(y[0], y[1]);
  } else if constexpr (N == 4) {
    // d03 = A y1 + B y3 = A (y1 + R y3), d12 = B y1 - A y3 = -A (y3 - R y1), R = B / A
    constexpr S A = S(K_A4X2), R = S(K_B4X2 / K_A4X2);
    const V s03 = add(y[0], y[2]), s12 = sub(y[0], y[2]);
    const V d03 = fmac(y[3], R, y[1]);
    const V d12 = fnmac(y[1], R, y[3]);
    x[0] = fmac(d03, A, s03);
    x[3] = fnmac(d03, A, s03);
    x[1] = fnmac(d12, A, s12);
    x[2] = fmac(d12, A, s12);
  } else {
    constexpr int H = N / 2;
    V ye[H], yo[H], u[H], v[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      ye[i] = y[2 * i];
      yo[i] = y[2 * i + 1];
    }
    idct2s<V, H>(ye, u);
    idct4s<V, H>(yo, v);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const S c = S(idct4_scale<H>(i));
      x[i] = fmac(v[i], c, u[i]);
      x[N - 1 - i] = fnmac(v[i], c, u[i]);
    }
  }
}

// inverse DCT-4 without the rotations' cosines (x[i] = idct4_scale<M>(i) * out[i]),
// gain sqrt(M): structure of reference _fastcore.pyx:155-185
template <typename V, int M>
DA_DEV void idct4s(const V (&y)[M], V (&x)[M]) {
  static_assert(M >= 4, "idct4s is only reached from idct2s with N >= 8");
  using S = typename Scalar<V>::type;
  constexpr int H = M / 2;
  constexpr int OFF = psi_off(M);
  constexpr S SQ2 = S(K_SQRT2);
  V c[H], sr[H], p[H], q[H];
  c[0] = mul(y[0], SQ2);
#pragma unroll
  for (int r = 1; r < H; ++r) {
    c[r] = add(y[2 * r], y[2 * r - 1]);
    sr[H - r] = sub(y[2 * r], y[2 * r - 1]);  // s[r-1], stored reversed
  }
  sr[0] = mul(y[2 * H - 1], -SQ2);            // s[H-1]
  idct2s<V, H>(c, p);
  // inverse DST2: reverse, inverse DCT2, sign-alternate (folded into the rotation)
  idct2s<V, H>(sr, q);
#pragma unroll
  for (int n = 0; n < H; ++n) {
    const S t = S(psi_s(OFF + n) / psi_c(OFF + n));
    if (n % 2 == 0) {  // cp (p - t q), cp (q + t p)
      x[n] = fnmac(q[n], t, p[n]);
      x[M - 1 - n] = fmac(p[n], t, q[n]);
    } else {           // cp (p + t q), -cp (q - t p)
      x[n] = fmac(q[n], t, p[n]);
      x[M - 1 - n] = fnmac(p[n], t, q[n]);
    }
  }
}

template <typename V, int M> DA_DEV void idct4p(const V (&y)[M], V (&x)[M]);
// DCT-3 (inverse DCT-2), gain sqrt(N), plain rotations (2 multiplies + 2 FMAs each):
// structure of reference _fastcore.pyx:120-152
template <typename V, int N>
DA_DEV void idct2p(const V (&y)[N], V (&x)[N]) {
  using S = typename Scalar<V>::type;
  if constexpr (N == 1) {
    x[0] = y[0];
  } else if constexpr (N == 2) {
    x[0] = add(y[0], y[1]);
    x[1] = sub(y[0], y[1]);
  } else if constexpr (N == 4) {
    constexpr S A = S(K_A4X2), B = S(K_B4X2);
    const V s03 = add(y[0], y[2]), s12 = sub(y[0], y[2]);
    const V d03 = fmac(y[1], A, mul(y[3], B));
    const V d12 = fnmac(y[3], A, mul(y[1], B));
    x[0] = add(s03, d03);
    x[3] = sub(s03, d03);
    x[1] = add(s12, d12);
    x[2] = sub(s12, d12);
  } else {
    constexpr int H = N / 2;
    V ye[H], yo[H], u[H], v[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      ye[i] = y[2 * i];
      yo[i] = y[2 * i + 1];
    }
    idct2p<V, H>(ye, u);
    idct4p<V, H>(yo, v);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      x[i] = add(u[i], v[i]);
      x[N - 1 - i] = sub(u[i], v[i]);
    }
  }
}

// inverse DCT-4, gain sqrt(M): structure of reference _fastcore.pyx:155-185
template <typename V, int M>
DA_DEV void idct4p(const V (&y)[M], V (&x)[M]) {
  static_assert(M >= 4, "idct4p is only reached from idct2p with N >= 8");
  using S = typename Scalar<V>::type;
  constexpr int H = M / 2;
  constexpr int OFF = psi_off(M);
  constexpr S SQ2 = S(K_SQRT2);
  V c[H], sr[H], p[H], q[H];
  c[0] = mul(y[0], SQ2);
#pragma unroll
  for (int r = 1; r < H; ++r) {
    c[r] = add(y[2 * r], y[2 * r - 1]);
    sr[H - r] = sub(y[2 * r], y[2 * r - 1]);  // s[r-1], stored reversed
  }
  sr[0] = mul(y[2 * H - 1], -SQ2);            // s[H-1]
  idct2p<V, H>(c, p);
  // inverse DST2: reverse, inverse DCT2, sign-alternate (folded into the rotation)
  idct2p<V, H>(sr, q);
#pragma unroll
  for (int n = 0; n < H; ++n) {
    const S cp = S(psi_c(OFF + n)), sp = S(psi_s(OFF + n));
    if (n % 2 == 0) {
      x[n] = fnmac(q[n], sp, mul(p[n], cp));
      x[M - 1 - n] = fmac(q[n], cp, mul(p[n], sp));
    } else {
      x[n] = fmac(q[n], sp, mul(p[n], cp));
      x[M - 1 - n] = fnmac(q[n], cp, mul(p[n], sp));
    }
  }
}


// Which form a kernel gets is a per-(type, size) choice, measured on the B200 (A/B
// libraries, profiles/r02_tuning.md): fp32 (scalar and packed) up to 32 points runs
// the scaled / deferred forms (fused round trips: config 2 +1.4 %, config 3 pre
// +5.6 %, post +1.5 %); fp64 (config 1: +4 % time) and the 64-point kernels (config
// 4's ring kernel: instruction-fetch stalls double, forward +3 %, inverse +12 %) keep
// the plain forms.  The choice depends on (type, size) only, never on the kernel
// family, so every kernel that computes the same transform stays bit-identical.
// DCTADJ_IDCT_SCALED / DCTADJ_DEFERRED = 0 build the plain forms everywhere.
#ifndef DCTADJ_IDCT_SCALED
#define DCTADJ_IDCT_SCALED 1
#endif
#ifndef DCTADJ_DEFERRED
#define DCTADJ_DEFERRED 1
#endif
#ifndef DCTADJ_SCALED_MAXN
#define DCTADJ_SCALED_MAXN 32
#endif
__host__ __device__ constexpr bool idct_scaled_policy(bool is_double, int n) {
  return DCTADJ_IDCT_SCALED != 0 && !is_double && n <= DCTADJ_SCALED_MAXN;
}
__host__ __device__ constexpr bool deferred_policy(bool is_double, int n) {
  return DCTADJ_DEFERRED != 0 && !is_double && n <= DCTADJ_SCALED_MAXN;
}
template <typename V, int N>
__host__ __device__ constexpr bool use_idct_scaled() {
  return idct_scaled_policy(std::is_same<V, double>::value, N);
}
template <typename S, int N>
__host__ __device__ constexpr bool use_deferred() {
  return deferred_policy(std::is_same<S, double>::value, N);
}

template <typename V, int N>
DA_DEV void idct2u(const V (&y)[N], V (&x)[N]) {
  if constexpr (use_idct_scaled<V, N>())
    idct2s<V, N>(y, x);
  else
    idct2p<V, N>(y, x);
}

// ---------------------------------------------------------------------------
// Per-axis stages (base stages unnormalized).  A 1-D adjusted transform on one axis is at most two
// stages (reference pipeline.py:176-191):
//   forward  PRE : [BAND|SUB|DENSE, base]      POST: [base, SUB|BAND|DENSE]
//   inverse  PRE : [base^-1, adj^T]            POST: [adj^T, base^-1]
// The host packs adj / adj^T (and the R*A*R flip for the DCT-8 pre variant) so
// the device only ever applies "the given coefficients".
enum Stage : int {
  ST_NONE = 0,
  ST_DCT2 = 1,   // dct2
  ST_IDCT2 = 2,  // idct2 (= DCT-3)
  ST_DST3 = 3,   // reverse -> idct2 -> negate odd
  ST_IDST3 = 4,  // negate odd -> dct2 -> reverse
  ST_BAND = 5,   // K-tap band, coefficients packed [N][2K-1]
  ST_SUB = 6,    // leading KxK block, coefficients packed [K][K]
  ST_DENSE = 7,  // full N x N from shared memory
  ST_GIVENS = 8, // (retired) the brick-wall layers in lifting form, 3 dependent FMAs each
  ST_GIVENS2 = 9, // K-tap band as K-1 brick-wall layers of plane rotations (reference
                  // design.py:225-243), scaled form: 2 FMAs each + one scale per sample
};

// Rotations in brick-wall layer l of an N-point band schedule (pairs (i, i+1),
// i = l%2, l%2 + 2, ...; reference design.py:234-243).
__host__ __device__ constexpr int givens_layer_rots(int n, int l) { return (n - (l % 2)) / 2; }
__host__ __device__ constexpr int givens_rots(int n, int k) {
  int r = 0;
  for (int l = 0; l < k - 1; ++l) r += givens_layer_rots(n, l);
  return r;
}

// op code = s1 | s2 << 4 | k << 8
__host__ __device__ constexpr int op_code(int s1, int s2 = ST_NONE, int k = 0) {
  return s1 | (s2 << 4) | (k << 8);
}
__host__ __device__ constexpr int op_s1(int c) { return c & 15; }
__host__ __device__ constexpr int op_s2(int c) { return (c >> 4) & 15; }
__host__ __device__ constexpr int op_k(int c) { return c >> 8; }

template <typename T, int N, int K, int S>
struct StageCoef {  // no coefficients
  static constexpr int count = 0;
};
template <typename T, int N, int K>
struct StageCoef<T, N, K, ST_BAND> {
  static constexpr int count = N * (2 * K - 1);
};
template <typename T, int N, int K>
struct StageCoef<T, N, K, ST_SUB> {
  static constexpr int count = K * K;
};
template <typename T, int N, int K>
struct StageCoef<T, N, K, ST_GIVENS2> {
  static constexpr int count = 2 * givens_rots(N, K) + N;  // (k1, k2) per rotation, N scales
};

template <typename T, int N, int CODE>
struct AxisOp {
  static constexpr int S1 = op_s1(CODE), S2 = op_s2(CODE), K = op_k(CODE);
  static constexpr int NC1 = StageCoef<T, N, K, S1>::count;
  static constexpr int NC2 = StageCoef<T, N, K, S2>::count;
  static_assert(NC1 == 0 || NC2 == 0, "at most one coefficient stage per axis");
  static constexpr int NCOEF = NC1 + NC2;
  static constexpr bool kDense = (S1 == ST_DENSE) || (S2 == ST_DENSE);
  static constexpr bool kIdentity = (S1 == ST_NONE) && (S2 == ST_NONE);
  // the base stages run unnormalized: gain sqrt(N) (removed once per launch) --
  // except behind a trailing scaled-Givens stage, whose per-sample scales carry
  // 1/sqrt(N) already (the host folds it in)
  static constexpr bool kBase = (S1 >= ST_DCT2 && S1 <= ST_IDST3) || (S2 >= ST_DCT2 && S2 <= ST_IDST3);
  static constexpr int kGainSq = (kBase && S2 != ST_GIVENS2) ? N : 1;  // gain^2
  // a forward-direction base (dct2 / idst3) in front of the scaled-rotation band runs
  // with deferred scales (dct2d): the band's input scales absorb them on the host
  static constexpr bool kDeferred =
      (S1 == ST_DCT2 || S1 == ST_IDST3) && S2 == ST_GIVENS2 && use_deferred<T, N>();
  // dct2 in front of the sub-block post-adjustment: the host folds the deferred scales of
  // the K adjusted inputs into the block's columns; the untouched tail is finalized
  static constexpr bool kDeferredSub = S1 == ST_DCT2 && S2 == ST_SUB && use_deferred<T, N>();
  struct Coef {
    T c[NCOEF > 0 ? NCOEF : 1];
  };
};

template <typename V, int N, int S, int K>
DA_DEV void run_stage(V (&v)[N], const typename Scalar<V>::type* __restrict__ cf,
                      const typename Scalar<V>::type* __restrict__ dense) {
  using Sc = typename Scalar<V>::type;
  if constexpr (S == ST_NONE) {
    return;
  } else if constexpr (S == ST_DCT2) {
    V y[N];
    if constexpr (use_deferred<Sc, N>()) {
      // deferred-scale form, finalized: one multiply per output whose scale is not 1
      // (186 + 30 instead of 242 at 32 points).  The sub-block post-adjustment below
      // (apply_axis) finalizes its untouched tail the same way, bit for bit.
      dct2d<V, ScUnit, N>(v, y);
      finalize_deferred<V, ScUnit, N, 0, false>(y, v);
    } else {
      dct2u<V, N>(v, y);
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = y[i];
    }
  } else if constexpr (S == ST_IDCT2) {
    V y[N];
    idct2u<V, N>(v, y);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = y[i];
  } else if constexpr (S == ST_DST3) {
    V r[N], y[N];
#pragma unroll
    for (int j = 0; j < N; ++j) r[j] = v[N - 1 - j];
    idct2u<V, N>(r, y);
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = (j % 2 == 0) ? y[j] : neg(y[j]);
  } else if constexpr (S == ST_IDST3) {
    V y[N];
    if constexpr (use_deferred<Sc, N>()) {
      dct2d<V, ScAlt, N>(v, y);  // the sign alternation is an input scale of -1
      finalize_deferred<V, ScAlt, N, 0, true>(y, v);
    } else {
      V a[N];
#pragma unroll
      for (int j = 0; j < N; ++j) a[j] = (j % 2 == 0) ? v[j] : neg(v[j]);
      dct2u<V, N>(a, y);
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = y[N - 1 - j];
    }
  } else if constexpr (S == ST_BAND) {
    constexpr int D = 2 * K - 1;
    V y[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      const int j0 = r - (K - 1) < 0 ? 0 : r - (K - 1);
      const int j1 = r + K > N ? N : r + K;
      V acc = mul(v[j0], cf[r * D + (j0 - r + K - 1)]);
#pragma unroll
      for (int j = j0 + 1; j < j1; ++j) acc = fmac(v[j], cf[r * D + (j - r + K - 1)], acc);
      y[r] = acc;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = y[i];
  } else if constexpr (S == ST_SUB) {
    static_assert(K <= N, "sub-block order exceeds transform size");
    V y[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      V acc = mul(v[0], cf[r * K]);
#pragma unroll
      for (int j = 1; j < K; ++j) acc = fmac(v[j], cf[r * K + j], acc);
      y[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < K; ++r) v[r] = y[r];
  } else if constexpr (S == ST_GIVENS2) {
    // y = L_{K-2} ... L_0 x, each layer index-disjoint rotations
    //   x_i' = c x_i - s x_j,  x_j' = s x_i + c x_j   (reference design.py:137-147)
    // with cos(theta) factored out and carried as a per-sample
    // scale: the held values are u = a U, v = b V (a, b known per sample), and
    //   U' = U + k1 V,  V' = V + k2 U,  k1 = -tan(theta) b / a,  k2 = tan(theta) a / b
    // (both scales times cos(theta)) -- 2 independent FMAs per rotation instead of
    // the lifting form's 3 dependent ones.  The host tracks the scales through the
    // schedule (|cos theta| >= 0.2, else the band runs another way) and appends
    // them; one multiply per sample at the end restores the rotated values.
#pragma unroll
    for (int l = 0; l < K - 1; ++l) {
#pragma unroll
      for (int i = l % 2; i + 1 < N; i += 2) {
        int q = 0;
#pragma unroll
        for (int m = 0; m < l; ++m) q += givens_layer_rots(N, m);
        q += (i - l % 2) / 2;
        const V u = v[i], w = v[i + 1];
        v[i] = fmac(w, cf[2 * q], u);
        v[i + 1] = fmac(u, cf[2 * q + 1], w);
      }
    }
    constexpr int R = givens_rots(N, K);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = mul(v[i], cf[2 * R + i]);
  } else if constexpr (S == ST_DENSE) {
    V y[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      V acc = mul(v[0], dense[r * N]);
#pragma unroll
      for (int j = 1; j < N; ++j) acc = fmac(v[j], dense[r * N + j], acc);
      y[r] = acc;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = y[i];
  }
}

// Output scales of the deferred base in front of a Givens stage (host side: the
// initial running scales of pack_givens2): v[j] = deferred_base_scale(...) * held[j].
template <int N, int S1>
__host__ __device__ constexpr double deferred_base_scale(int j) {
  return S1 == ST_IDST3 ? dct2d_out_scale<N, true>(N - 1 - j) : dct2d_out_scale<N, false>(j);
}

template <typename V, int N, int CODE>
DA_DEV void apply_axis(V (&v)[N],
                       const typename AxisOp<typename Scalar<V>::type, N, CODE>::Coef& cf,
                       const typename Scalar<V>::type* __restrict__ dense) {
  using Op = AxisOp<typename Scalar<V>::type, N, CODE>;
  if constexpr (Op::kDeferredSub) {
    constexpr int K = Op::K;
    V y[N];
    dct2d<V, ScUnit, N>(v, y);
#pragma unroll
    for (int r = 0; r < K; ++r) {  // cf = block * diag(scale_0..K-1): acts on the held values
      V acc = mul(y[0], cf.c[r * K]);
#pragma unroll
      for (int j = 1; j < K; ++j) acc = fmac(y[j], cf.c[r * K + j], acc);
      v[r] = acc;
    }
    finalize_deferred<V, ScUnit, N, K, false>(y, v);
    return;
  } else if constexpr (Op::kDeferred) {
    V y[N];
    if constexpr (Op::S1 == ST_IDST3) {  // negate odd (in the scales) -> dct2 -> reverse
      dct2d<V, ScAlt, N>(v, y);
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = y[N - 1 - j];
    } else {
      dct2d<V, ScUnit, N>(v, y);
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = y[j];
    }
  } else {
    run_stage<V, N, Op::S1, Op::K>(v, cf.c, dense);
  }
  run_stage<V, N, Op::S2, Op::K>(v, cf.c, dense);
}

}  // namespace dctadj

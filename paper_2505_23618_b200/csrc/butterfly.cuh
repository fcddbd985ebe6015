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
#pragma once
#include <cstdint>

#include "twiddles.h"

namespace dctadj {

#define DA_DEV __device__ __forceinline__

// Unnormalized recursion.  The reference scales by 1/sqrt(2) at every level
// (u = (a+b)/sqrt2, v = (a-b)/sqrt2, and (c +- s)/sqrt2 in the DCT-4 output
// butterflies): ~125 of the 411 flops of a 32-point DCT-2.  Dropping those
// scalings makes every routine below return sqrt(N) x the orthonormal result,
// uniformly over its outputs (induction: dct2u_N = sqrt2 * {dct2u_N/2, dct4u_N/2}
// needs g(dct2u_M) == g(dct4u_M); the bases give g = 2 at M = 4, and dct4u only
// needs its two unscaled outputs y[0], y[M-1] multiplied by sqrt2).  The gain is
// removed once per launch (1/32 for a 32x32 block, exact in binary).
template <typename T, int N> DA_DEV void dct2u(const T (&x)[N], T (&y)[N]);
template <typename T, int M> DA_DEV void dct4u(const T (&x)[M], T (&y)[M]);
template <typename T, int N> DA_DEV void idct2u(const T (&y)[N], T (&x)[N]);
template <typename T, int M> DA_DEV void idct4u(const T (&y)[M], T (&x)[M]);

// DCT-2, gain sqrt(N): structure of reference _fastcore.pyx:50-84
template <typename T, int N>
DA_DEV void dct2u(const T (&x)[N], T (&y)[N]) {
  if constexpr (N == 1) {
    y[0] = x[0];
  } else if constexpr (N == 2) {
    y[0] = x[0] + x[1];
    y[1] = x[0] - x[1];
  } else if constexpr (N == 4) {
    constexpr T A = T(K_A4X2), B = T(K_B4X2);
    const T s03 = x[0] + x[3], d03 = x[0] - x[3];
    const T s12 = x[1] + x[2], d12 = x[1] - x[2];
    y[0] = s03 + s12;
    y[2] = s03 - s12;
    y[1] = A * d03 + B * d12;
    y[3] = B * d03 - A * d12;
  } else {
    constexpr int H = N / 2;
    T u[H], v[H], eu[H], ov[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const T a = x[i], b = x[N - 1 - i];
      u[i] = a + b;
      v[i] = a - b;
    }
    dct2u<T, H>(u, eu);
    dct4u<T, H>(v, ov);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      y[2 * i] = eu[i];
      y[2 * i + 1] = ov[i];
    }
  }
}

// DCT-4, gain sqrt(M): structure of reference _fastcore.pyx:87-117
template <typename T, int M>
DA_DEV void dct4u(const T (&x)[M], T (&y)[M]) {
  static_assert(M >= 4, "dct4u is only reached from dct2u with N >= 8");
  constexpr int H = M / 2;
  constexpr int OFF = psi_off(M);
  constexpr T SQ2 = T(K_SQRT2);
  T p[H], sq[H], c[H], s2[H];
#pragma unroll
  for (int n = 0; n < H; ++n) {
    const T a = x[n], b = x[M - 1 - n];
    const T cp = T(psi_c(OFF + n)), sp = T(psi_s(OFF + n));
    p[n] = a * cp + b * sp;
    const T q = b * cp - a * sp;
    // DST2(q) = reverse(DCT2(sign-alternated q))
    sq[n] = (n % 2 == 0) ? q : -q;
  }
  dct2u<T, H>(p, c);
  dct2u<T, H>(sq, s2);
  y[0] = SQ2 * c[0];
#pragma unroll
  for (int r = 1; r < H; ++r) {
    y[2 * r] = c[r] + s2[H - r];
    y[2 * r - 1] = c[r] - s2[H - r];
  }
  y[2 * H - 1] = -SQ2 * s2[0];
}

// DCT-3 (inverse DCT-2), gain sqrt(N): structure of reference _fastcore.pyx:120-152
template <typename T, int N>
DA_DEV void idct2u(const T (&y)[N], T (&x)[N]) {
  if constexpr (N == 1) {
    x[0] = y[0];
  } else if constexpr (N == 2) {
    x[0] = y[0] + y[1];
    x[1] = y[0] - y[1];
  } else if constexpr (N == 4) {
    constexpr T A = T(K_A4X2), B = T(K_B4X2);
    const T s03 = y[0] + y[2], s12 = y[0] - y[2];
    const T d03 = A * y[1] + B * y[3];
    const T d12 = B * y[1] - A * y[3];
    x[0] = s03 + d03;
    x[3] = s03 - d03;
    x[1] = s12 + d12;
    x[2] = s12 - d12;
  } else {
    constexpr int H = N / 2;
    T ye[H], yo[H], u[H], v[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      ye[i] = y[2 * i];
      yo[i] = y[2 * i + 1];
    }
    idct2u<T, H>(ye, u);
    idct4u<T, H>(yo, v);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      x[i] = u[i] + v[i];
      x[N - 1 - i] = u[i] - v[i];
    }
  }
}

// inverse DCT-4, gain sqrt(M): structure of reference _fastcore.pyx:155-185
template <typename T, int M>
DA_DEV void idct4u(const T (&y)[M], T (&x)[M]) {
  static_assert(M >= 4, "idct4u is only reached from idct2u with N >= 8");
  constexpr int H = M / 2;
  constexpr int OFF = psi_off(M);
  constexpr T SQ2 = T(K_SQRT2);
  T c[H], sr[H], p[H], q[H];
  c[0] = SQ2 * y[0];
#pragma unroll
  for (int r = 1; r < H; ++r) {
    c[r] = y[2 * r] + y[2 * r - 1];
    sr[H - r] = y[2 * r] - y[2 * r - 1];  // s[r-1], stored reversed
  }
  sr[0] = -SQ2 * y[2 * H - 1];            // s[H-1]
  idct2u<T, H>(c, p);
  // inverse DST2: reverse, inverse DCT2, sign-alternate
  idct2u<T, H>(sr, q);
#pragma unroll
  for (int n = 0; n < H; ++n) {
    const T qn = (n % 2 == 0) ? q[n] : -q[n];
    const T cp = T(psi_c(OFF + n)), sp = T(psi_s(OFF + n));
    x[n] = p[n] * cp - qn * sp;
    x[M - 1 - n] = p[n] * sp + qn * cp;
  }
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
};

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

template <typename T, int N, int CODE>
struct AxisOp {
  static constexpr int S1 = op_s1(CODE), S2 = op_s2(CODE), K = op_k(CODE);
  static constexpr int NC1 = StageCoef<T, N, K, S1>::count;
  static constexpr int NC2 = StageCoef<T, N, K, S2>::count;
  static_assert(NC1 == 0 || NC2 == 0, "at most one coefficient stage per axis");
  static constexpr int NCOEF = NC1 + NC2;
  static constexpr bool kDense = (S1 == ST_DENSE) || (S2 == ST_DENSE);
  static constexpr bool kIdentity = (S1 == ST_NONE) && (S2 == ST_NONE);
  // the base stages run unnormalized: gain sqrt(N) (removed once per launch)
  static constexpr bool kBase = (S1 >= ST_DCT2 && S1 <= ST_IDST3) || (S2 >= ST_DCT2 && S2 <= ST_IDST3);
  static constexpr int kGainSq = kBase ? N : 1;  // gain^2
  struct Coef {
    T c[NCOEF > 0 ? NCOEF : 1];
  };
};

template <typename T, int N, int S, int K>
DA_DEV void run_stage(T (&v)[N], const T* __restrict__ cf, const T* __restrict__ dense) {
  if constexpr (S == ST_NONE) {
    return;
  } else if constexpr (S == ST_DCT2) {
    T y[N];
    dct2u<T, N>(v, y);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = y[i];
  } else if constexpr (S == ST_IDCT2) {
    T y[N];
    idct2u<T, N>(v, y);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = y[i];
  } else if constexpr (S == ST_DST3) {
    T r[N], y[N];
#pragma unroll
    for (int j = 0; j < N; ++j) r[j] = v[N - 1 - j];
    idct2u<T, N>(r, y);
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = (j % 2 == 0) ? y[j] : -y[j];
  } else if constexpr (S == ST_IDST3) {
    T a[N], y[N];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = (j % 2 == 0) ? v[j] : -v[j];
    dct2u<T, N>(a, y);
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = y[N - 1 - j];
  } else if constexpr (S == ST_BAND) {
    constexpr int D = 2 * K - 1;
    T y[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      T acc = T(0);
      bool first = true;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int j = r - (K - 1) + d;
        if (j >= 0 && j < N) {
          if (first) {
            acc = cf[r * D + d] * v[j];
            first = false;
          } else {
            acc = fma(cf[r * D + d], v[j], acc);
          }
        }
      }
      y[r] = acc;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = y[i];
  } else if constexpr (S == ST_SUB) {
    static_assert(K <= N, "sub-block order exceeds transform size");
    T y[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      T acc = cf[r * K] * v[0];
#pragma unroll
      for (int j = 1; j < K; ++j) acc = fma(cf[r * K + j], v[j], acc);
      y[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < K; ++r) v[r] = y[r];
  } else if constexpr (S == ST_DENSE) {
    // dense rows are read as 16-byte broadcasts from shared memory
    T y[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      T acc = dense[r * N] * v[0];
#pragma unroll
      for (int j = 1; j < N; ++j) acc = fma(dense[r * N + j], v[j], acc);
      y[r] = acc;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = y[i];
  }
}

template <typename T, int N, int CODE>
DA_DEV void apply_axis(T (&v)[N], const typename AxisOp<T, N, CODE>::Coef& cf,
                       const T* __restrict__ dense) {
  using Op = AxisOp<T, N, CODE>;
  run_stage<T, N, Op::S1, Op::K>(v, cf.c, dense);
  run_stage<T, N, Op::S2, Op::K>(v, cf.c, dense);
}

}  // namespace dctadj

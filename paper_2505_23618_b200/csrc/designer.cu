// designer.cu -- the adjustment designer's cyclic coordinate descent on the GPU
// (designer acceleration; off the transform path).
//
// Restates reference design.py:377-543 (_CoordinateDescent.run, the eps = None
// path used by optimize_adjustment) with every random restart in its own CTA:
// the composed-error matrix E = H - D, the adjustment A and the partial
// products (UA, VA, and UW or VW) live in shared memory (fp64, N <= 64), and
// each angle step is
//   8 length-N reductions + 2 matrix-vector products (the degree-2 trig
//   polynomial of the weighted error in (cos, sin), design.py:442-475)
//   -> the 33-point grid (one lane per point), golden-section refinement to
//      1e-12 and the {0, theta_old} candidates with the reference's tie rule
//      (design.py:333-374) in the reference's order
//   -> rank-2 updates of E and A (design.py:503-510)
//   -> strip the next rotation from UA (UW), apply this one to VA (VW)
//      (design.py:515-523).
// Results agree with the reference up to floating-point reduction order (the
// reference sums with BLAS / numpy); the host (design.py) merges restarts and
// builds the record exactly as optimize_adjustment does (design.py:560-613).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/dctadj.h"
#include "launch.cuh"

namespace dctadj {
namespace designer {

constexpr int kMaxN = 64;
constexpr int kThreads = 256;
constexpr int kGrid = 33;               // reference _SEARCH_GRID
constexpr double kAngleTol = 1e-12;     // reference _ANGLE_TOL
constexpr double kGolden = 0.6180339887498949;  // reference _GOLDEN = (sqrt5 - 1) / 2
constexpr double kHalfPi = 1.5707963267948966;

struct Args {
  int n, m, side;  // side: 0 = PRE (H = B A), 1 = POST (H = A B)
  const double* base;     // n x n
  const double* desired;  // n x n
  const double* w;        // n frequency weights
  const int* rp;          // m
  const int* rq;          // m
  const double* theta0;   // restarts x m
  int max_sweeps;
  double tol;
  double* theta;          // restarts x m (out)
  double* trace;          // restarts x (max_sweeps + 1) (out)
  int* sweeps;            // restarts (out): trace length - 1
  int* converged;         // restarts (out)
};

// block-wide sum of one value per thread (all threads must call)
__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kThreads / 32; ++k) s += red[k];
  return s;
}

// m[p,:], m[q,:] <- c rp - s rq, s rp + c rq  (design.py:317-321); threads j < n
__device__ void apply_rows(double* mat, int n, int p, int q, double c, double s) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double a = mat[p * n + j], b = mat[q * n + j];
    mat[p * n + j] = c * a - s * b;
    mat[q * n + j] = s * a + c * b;
  }
}
// m[:,p], m[:,q] <- c cp - s cq, s cp + c cq  (design.py:324-330)
__device__ void strip_cols(double* mat, int n, int p, int q, double c, double s) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = mat[i * n + p], b = mat[i * n + q];
    mat[i * n + p] = c * a - s * b;
    mat[i * n + q] = s * a + c * b;
  }
}

struct Quad {  // the weighted error as a degree-2 polynomial in (cos, sin)
  double cst, bp, bq, app, aqq, apq;
  __device__ double operator()(double c, double s) const {
    return cst + 2 * c * bp + 2 * s * bq + c * c * app + s * s * aqq + 2 * c * s * apq;
  }
  __device__ double at(double th) const {
    double s, c;
    sincos(th, &s, &c);
    return (*this)(c, s);
  }
};

// reference _golden_min (design.py:333-347) on a whole warp, speculatively:
// the points a golden-section
// step creates depend only on the earlier steps' comparisons, so each round
// evaluates every point of the next 5 steps' decision tree at once (31 lanes,
// heap order: node k's children are 2k (f1 <= f2: the bracket keeps [a, x2])
// and 2k+1), then replays the 5 comparisons on the values.  Points, values and
// decisions are the serial ones bit for bit; the dependent sincos chain drops
// from ~56 to ~12 links.  All 32 lanes call; every lane returns the result.
struct GoldenState {
  double a, b, x1, x2;
  // one step taking branch `keep_left` (f1 <= f2); returns the new point
  __device__ double step(bool keep_left) {
    if (keep_left) {
      b = x2;
      x2 = x1;
      x1 = b - kGolden * (b - a);
      return x1;
    }
    a = x1;
    x1 = x2;
    x2 = a + kGolden * (b - a);
    return x2;
  }
};

__device__ double golden_min_warp(const Quad& f, double lo, double hi, int lane) {
  constexpr int kDepth = 5;  // 2^5 - 1 = 31 tree nodes per round
  GoldenState st{lo, hi, 0.0, 0.0};
  st.x1 = hi - kGolden * (hi - lo);
  st.x2 = lo + kGolden * (hi - lo);
  const double fx = f.at(lane == 0 ? st.x1 : st.x2);
  double f1 = __shfl_sync(0xffffffffu, fx, 0), f2 = __shfl_sync(0xffffffffu, fx, 1);
  while (st.b - st.a > kAngleTol) {
    // lane L evaluates tree node L + 1: the first decision is known, the next
    // ones are the bits of the node number below its leading one
    const int node = lane + 1;
    const int depth = 31 - __clz(node);  // node's level - 1
    GoldenState sp = st;
    double pt = sp.step(f1 <= f2);
    for (int d = depth - 1; d >= 0; --d) pt = sp.step(((node >> d) & 1) == 0);
    const double val = lane < 31 ? f.at(pt) : 0.0;
    // replay the real path through the tree
    int k = 1;
    for (int lvl = 0; lvl < kDepth && st.b - st.a > kAngleTol; ++lvl) {
      const bool keep_left = f1 <= f2;
      if (lvl > 0) k = 2 * k + (keep_left ? 0 : 1);
      st.step(keep_left);
      const double v = __shfl_sync(0xffffffffu, val, k - 1);
      if (keep_left) {
        f2 = f1;
        f1 = v;
      } else {
        f1 = f2;
        f2 = v;
      }
    }
  }
  return 0.5 * (st.a + st.b);
}

// one CTA = one restart
__global__ void __launch_bounds__(kThreads) cd_kernel(const Args g) {
  extern __shared__ double sm[];
  const int n = g.n, nn = n * n, m = g.m, tid = threadIdx.x;
  const bool pre = g.side == 0;
  double* E = sm;          // composed error H - D
  double* A = E + nn;      // adjustment
  double* UA = A + nn;     // left partial product of A (rotation t stripped)
  double* VA = UA + nn;    // right partial product of A
  double* X = VA + nn;     // PRE: UW (left factor of H);  POST: VW (right factor)
  double* w = X + nn;      // n
  double* vec = w + kMaxN; // 4 x n scratch: up, uq, vp, vq
  double* ev = vec + 4 * kMaxN;  // 2 x n: E vp, E vq
  double* th = ev + 2 * kMaxN;   // m angles
  double* red = th + m;          // kThreads / 32
  __shared__ double sc[8];       // broadcast scalars
  const int r = blockIdx.x;
  const double* base = g.base;
  const double* des = g.desired;

  for (int i = tid; i < n; i += kThreads) w[i] = g.w[i];
  for (int t = tid; t < m; t += kThreads) th[t] = g.theta0[static_cast<size_t>(r) * m + t];
  // A = realize(theta) (design.py:421-425)
  for (int e = tid; e < nn; e += kThreads) A[e] = (e / n == e % n) ? 1.0 : 0.0;
  __syncthreads();
  for (int t = 0; t < m; ++t) {
    double s, c;
    sincos(th[t], &s, &c);
    apply_rows(A, n, g.rp[t], g.rq[t], c, s);
    __syncthreads();
  }
  // E = compose(A) - D; wobj = sum_i w_i sum_j E_ij^2
  double part = 0.0;
  for (int e = tid; e < nn; e += kThreads) {
    const int i = e / n, j = e % n;
    double h = 0.0;
    if (pre)
      for (int k = 0; k < n; ++k) h += base[i * n + k] * A[k * n + j];
    else
      for (int k = 0; k < n; ++k) h += A[i * n + k] * base[k * n + j];
    const double d = h - des[e];
    E[e] = d;
    part += w[i] * d * d;
  }
  double wobj = block_sum(part, red);
  double obj = wobj;
  double* trace = g.trace + static_cast<size_t>(r) * (g.max_sweeps + 1);
  if (tid == 0) trace[0] = obj;
  int sweeps = 0, converged = 0;
  if (m == 0) converged = 1;

  for (int sweep = 0; sweep < g.max_sweeps && m > 0; ++sweep) {
    // partial products around rotation 0 (design.py:437-449)
    {
      double s0, c0;
      sincos(th[0], &s0, &c0);
      for (int e = tid; e < nn; e += kThreads) {
        UA[e] = A[e];
        VA[e] = (e / n == e % n) ? 1.0 : 0.0;
        X[e] = pre ? E[e] + des[e] : base[e];  // PRE: UW = H;  POST: VW = B
      }
      __syncthreads();
      strip_cols(UA, n, g.rp[0], g.rq[0], c0, s0);
      if (pre) strip_cols(X, n, g.rp[0], g.rq[0], c0, s0);
      __syncthreads();
    }
    // POST: UW aliases UA; PRE: VW aliases VA
    const double* UW = pre ? X : UA;
    const double* VW = pre ? VA : X;
    for (int t = 0; t < m; ++t) {
      const int p = g.rp[t], q = g.rq[t];
      double so, co;
      sincos(th[t], &so, &co);
      for (int i = tid; i < n; i += kThreads) {
        vec[i] = UW[i * n + p];
        vec[kMaxN + i] = UW[i * n + q];
        vec[2 * kMaxN + i] = VW[p * n + i];
        vec[3 * kMaxN + i] = VW[q * n + i];
      }
      __syncthreads();
      // E vp, E vq: 4 threads per row (whole warps take part in the shuffles)
      if ((tid & ~31) < 4 * n) {
        const int k = tid, i = k >> 2, part4 = k & 3;
        const bool act = k < 4 * n;
        double a0 = 0.0, a1 = 0.0;
        if (act)
          for (int j = part4; j < n; j += 4) {
            a0 += E[i * n + j] * vec[2 * kMaxN + j];
            a1 += E[i * n + j] * vec[3 * kMaxN + j];
          }
        a0 += __shfl_xor_sync(0xffffffffu, a0, 1);
        a0 += __shfl_xor_sync(0xffffffffu, a0, 2);
        a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
        a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
        if (act && part4 == 0) {
          ev[i] = a0;
          ev[kMaxN + i] = a1;
        }
      }
      __syncthreads();
      // the ten length-n sums, one warp each (n <= 64: two elements per lane)
      {
        const int warp = tid >> 5, lane = tid & 31;
        double acc = 0.0;
        for (int i = lane; i < n; i += 32) {
          const double up = vec[i], uq = vec[kMaxN + i], vp = vec[2 * kMaxN + i],
                       vq = vec[3 * kMaxN + i], wi = w[i];
          switch (warp) {
            case 0: acc += wi * up * up; break;             // suu_pp
            case 1: acc += wi * uq * uq; break;             // suu_qq
            case 2: acc += wi * up * uq; break;             // suu_pq
            case 3: acc += vp * vp; break;                  // svv_pp
            case 4: acc += vq * vq; break;                  // svv_qq
            case 5: acc += vp * vq; break;                  // svv_pq
            case 6: acc += wi * (up * ev[i] + uq * ev[kMaxN + i]); break;  // we_p
            case 7: acc += wi * (uq * ev[i] - up * ev[kMaxN + i]); break;  // we_q
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) red[warp] = acc;
      }
      __syncthreads();
      if (tid < 32) {  // warp 0: the 1-D minimisation (design.py:352-374)
        const int lane = tid;
        const double suu_pp = red[0], suu_qq = red[1], suu_pq = red[2];
        const double svv_pp = red[3], svv_qq = red[4], svv_pq = red[5];
        const double we_p = red[6], we_q = red[7];
        Quad f;
        f.app = suu_pp * svv_pp + 2 * suu_pq * svv_pq + suu_qq * svv_qq;
        f.aqq = suu_qq * svv_pp - 2 * suu_pq * svv_pq + suu_pp * svv_qq;
        f.apq = (suu_pq * svv_pp - suu_pp * svv_pq + suu_qq * svv_pq - suu_pq * svv_qq);
        f.bp = we_p - co * f.app - so * f.apq;
        f.bq = we_q - co * f.apq - so * f.aqq;
        f.cst = (wobj - 2 * co * we_p - 2 * so * we_q + co * co * f.app + so * so * f.aqq +
                 2 * co * so * f.apq);
        // the 33 grid values, one (lane 0: two) per lane; argmin keeps the first
        // minimum like np.argmin.  Lanes 1 / 2 also evaluate the two candidates.
        const double step = 2 * kHalfPi / (kGrid - 1);
        double gbest = f.at(-kHalfPi + lane * step);
        int kbest = lane;
        if (lane == 0) {
          const double g32 = f.at(-kHalfPi + (kGrid - 1) * step);
          if (g32 < gbest) {
            gbest = g32;
            kbest = kGrid - 1;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double gv = __shfl_xor_sync(0xffffffffu, gbest, o);
          const int gk = __shfl_xor_sync(0xffffffffu, kbest, o);
          if (gv < gbest || (gv == gbest && gk < kbest)) {
            gbest = gv;
            kbest = gk;
          }
        }
        const double th_old = th[t];
        const double fcand = lane == 1 ? f.at(0.0) : lane == 2 ? f.at(th_old) : 0.0;
        const double fc0 = __shfl_sync(0xffffffffu, fcand, 1);
        const double fco = __shfl_sync(0xffffffffu, fcand, 2);
        const double gk = -kHalfPi + kbest * step;
        const double lo = fmax(-kHalfPi, gk - step), hi = fmin(kHalfPi, gk + step);
        const double t_gold = golden_min_warp(f, lo, hi, lane);
        if (lane == 0) {
          double t_best = t_gold;
          double f_best = f.at(t_best);
          const double cands[2] = {0.0, th_old}, fcs[2] = {fc0, fco};
          for (int ci = 0; ci < 2; ++ci) {
            const double fc = fcs[ci];
            const double tie = 1e-15 * (1.0 + fabs(f_best));
            if (fc < f_best - tie ||
                (fabs(fc - f_best) <= tie && fabs(cands[ci]) < fabs(t_best))) {
              f_best = fc;
              t_best = cands[ci];
            }
          }
          double sn, cn;
          sincos(t_best, &sn, &cn);
          sc[0] = cn;
          sc[1] = sn;
          sc[2] = f_best;
          sc[3] = f(cn, sn);  // the new weighted objective
          th[t] = t_best;
        }
      }
      __syncthreads();
      const double cn = sc[0], sn = sc[1], dc = cn - co, ds = sn - so;
      obj = sc[2];
      wobj = sc[3];
      // rank-2 updates (design.py:503-510); UA / VA are read before they change
      for (int e = tid; e < nn; e += kThreads) {
        const int i = e / n, j = e % n;
        const double up = vec[i], uq = vec[kMaxN + i], vp = vec[2 * kMaxN + j],
                     vq = vec[3 * kMaxN + j];
        E[e] += up * (dc * vp - ds * vq) + uq * (dc * vq + ds * vp);
        const double ap = UA[i * n + p], aq = UA[i * n + q];
        const double bp = VA[p * n + j], bq = VA[q * n + j];
        A[e] += ap * (dc * bp - ds * bq) + aq * (dc * bq + ds * bp);
      }
      __syncthreads();
      if (t + 1 < m) {  // design.py:515-523
        const int pn = g.rp[t + 1], qn = g.rq[t + 1];
        double s1, c1;
        sincos(th[t + 1], &s1, &c1);
        strip_cols(UA, n, pn, qn, c1, s1);
        if (pre) strip_cols(X, n, pn, qn, c1, s1);
        apply_rows(VA, n, p, q, cn, sn);
        if (!pre) apply_rows(X, n, p, q, cn, sn);
        __syncthreads();
      }
    }
    ++sweeps;
    const double prev = trace[sweeps - 1];
    __syncthreads();
    if (tid == 0) trace[sweeps] = obj;
    if (prev - obj < g.tol * (1.0 + fabs(obj))) {
      converged = 1;
      break;
    }
  }
  for (int t = tid; t < m; t += kThreads) g.theta[static_cast<size_t>(r) * m + t] = th[t];
  if (tid == 0) {
    g.sweeps[r] = sweeps;
    g.converged[r] = converged;
  }
}

}  // namespace designer
}  // namespace dctadj

using namespace dctadj;

extern "C" int dctadj_design_cd(int32_t n, const double* base, const double* desired,
                                const double* weights, int32_t side, int32_t m, const int32_t* rp,
                                const int32_t* rq, int32_t restarts, const double* theta0,
                                int32_t max_sweeps, double tol, double* theta_out,
                                double* trace_out, int32_t* sweeps_out, int32_t* converged_out,
                                int32_t device) {
  using namespace designer;
  if (n < 1 || n > kMaxN) {
    set_last_error("designer: size %d outside 1..%d", n, kMaxN);
    return ST_ERR_DIMENSION;
  }
  if (side != 0 && side != 1) {
    set_last_error("designer: side must be 0 (pre) or 1 (post), got %d", side);
    return ST_ERR_VALUE;
  }
  if (m < 0 || restarts < 1 || max_sweeps < 1 || !(tol > 0)) {
    set_last_error("designer: bad m=%d restarts=%d max_sweeps=%d tol=%g", m, restarts, max_sweeps,
                   tol);
    return ST_ERR_VALUE;
  }
  if (!base || !desired || !weights || !theta_out || !trace_out || !sweeps_out ||
      !converged_out || (m > 0 && (!rp || !rq || !theta0))) {
    set_last_error("designer: NULL argument");
    return ST_ERR_VALUE;
  }
  for (int t = 0; t < m; ++t)
    if (rp[t] < 0 || rp[t] >= n || rq[t] < 0 || rq[t] >= n || rp[t] == rq[t]) {
      set_last_error("designer: rotation %d pairs (%d, %d) outside an %d-point transform", t,
                     rp[t], rq[t], n);
      return ST_ERR_VALUE;
    }
  const size_t smem = sizeof(double) * (5 * n * n + 7 * kMaxN + m + kThreads / 32);
  if (smem > 227 * 1024) {
    set_last_error("designer: %d rotations do not fit shared memory", m);
    return ST_ERR_VALUE;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    set_last_error("designer: cudaSetDevice(%d) failed", device);
    return ST_ERR_CUDA;
  }
  const size_t nn = static_cast<size_t>(n) * n, tr = static_cast<size_t>(restarts) * (max_sweeps + 1);
  double *d_base = nullptr, *d_des = nullptr, *d_w = nullptr, *d_t0 = nullptr, *d_th = nullptr,
         *d_tr = nullptr;
  int *d_rp = nullptr, *d_rq = nullptr, *d_sw = nullptr, *d_cv = nullptr;
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  ok(cudaMalloc(&d_base, nn * 8));
  ok(cudaMalloc(&d_des, nn * 8));
  ok(cudaMalloc(&d_w, n * 8));
  ok(cudaMalloc(&d_t0, static_cast<size_t>(restarts) * (m ? m : 1) * 8));
  ok(cudaMalloc(&d_th, static_cast<size_t>(restarts) * (m ? m : 1) * 8));
  ok(cudaMalloc(&d_tr, tr * 8));
  ok(cudaMalloc(&d_rp, (m ? m : 1) * 4));
  ok(cudaMalloc(&d_rq, (m ? m : 1) * 4));
  ok(cudaMalloc(&d_sw, restarts * 4));
  ok(cudaMalloc(&d_cv, restarts * 4));
  ok(cudaMemcpy(d_base, base, nn * 8, cudaMemcpyHostToDevice));
  ok(cudaMemcpy(d_des, desired, nn * 8, cudaMemcpyHostToDevice));
  ok(cudaMemcpy(d_w, weights, n * 8, cudaMemcpyHostToDevice));
  if (m > 0) {
    ok(cudaMemcpy(d_t0, theta0, static_cast<size_t>(restarts) * m * 8, cudaMemcpyHostToDevice));
    ok(cudaMemcpy(d_rp, rp, m * 4, cudaMemcpyHostToDevice));
    ok(cudaMemcpy(d_rq, rq, m * 4, cudaMemcpyHostToDevice));
  }
  ok(cudaMemset(d_tr, 0, tr * 8));
  if (e == cudaSuccess) {
    Args a{n, m, side, d_base, d_des, d_w, d_rp, d_rq, d_t0, max_sweeps, tol, d_th, d_tr, d_sw, d_cv};
    ok(cudaFuncSetAttribute(cd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cd_kernel<<<restarts, kThreads, smem>>>(a);
    ok(cudaGetLastError());
    ok(cudaDeviceSynchronize());
  }
  if (m > 0) ok(cudaMemcpy(theta_out, d_th, static_cast<size_t>(restarts) * m * 8, cudaMemcpyDeviceToHost));
  ok(cudaMemcpy(trace_out, d_tr, tr * 8, cudaMemcpyDeviceToHost));
  ok(cudaMemcpy(sweeps_out, d_sw, restarts * 4, cudaMemcpyDeviceToHost));
  ok(cudaMemcpy(converged_out, d_cv, restarts * 4, cudaMemcpyDeviceToHost));
  for (void* p : {(void*)d_base, (void*)d_des, (void*)d_w, (void*)d_t0, (void*)d_th, (void*)d_tr,
                  (void*)d_rp, (void*)d_rq, (void*)d_sw, (void*)d_cv})
    if (p) cudaFree(p);
  if (e != cudaSuccess) {
    set_last_error("designer: %s", cudaGetErrorString(e));
    return ST_ERR_CUDA;
  }
  return ST_OK;
}

// givens_pack.h -- host-side packing of a brick-wall Givens schedule for the
// scaled-rotation band stage (ST_GIVENS2, butterfly.cuh).  Host only; shared by
// abi.cu and the CPU unit test of the butterflies (tests/butterfly_host.cpp).
//
// Coefficients in application order -- layers 0..K-2 forward; for A^T the layers
// reversed with negated angles (for even K they keep the l%2 offsets): per
// rotation (k1, k2) = (-t b / a, t a / b) with t = tan(theta) and a, b the running
// scales of the pair, then the n final scales (times `gain` when the stage trails
// the base: its 1/sqrt(n) is folded in).  When the stage trails a deferred-scale
// base (dct2d: base_before = ST_DCT2 or ST_IDST3) the running scales start from
// that base's output scales instead of 1, which is what makes the deferral free.
// false when some |cos(theta)| < kGivens2MinCos (large tan: the band then runs as
// the matrix product or the dense composite).
#pragma once
#include <cmath>
#include <vector>

#include "butterfly.cuh"

namespace dctadj {

constexpr double kGivens2MinCos = 0.2;

// scale of sample j after the deferred-scale base that precedes a trailing Givens stage
template <int S1>
inline double deferred_scale_of(int n, int j) {
  switch (n) {
    case 4: return deferred_base_scale<4, S1>(j);
    case 8: return deferred_base_scale<8, S1>(j);
    case 16: return deferred_base_scale<16, S1>(j);
    case 32: return deferred_base_scale<32, S1>(j);
    case 64: return deferred_base_scale<64, S1>(j);
    default: return 1.0;
  }
}

inline bool pack_givens2(int n, int k, const double* givens, bool inverse, double gain,
                         int base_before, std::vector<double>& c) {
  std::vector<int> start(k, 0);
  for (int l = 0; l + 1 < k; ++l) start[l + 1] = start[l] + givens_layer_rots(n, l);
  std::vector<double> a(static_cast<size_t>(n), 1.0);
  for (int j = 0; j < n; ++j)
    a[j] = base_before == ST_IDST3  ? deferred_scale_of<ST_IDST3>(n, j)
           : base_before == ST_DCT2 ? deferred_scale_of<ST_DCT2>(n, j)
                                    : 1.0;
  c.clear();
  for (int s = 0; s < k - 1; ++s) {
    const int l = inverse ? k - 2 - s : s;
    for (int r = 0; r < givens_layer_rots(n, l); ++r) {
      const double th = inverse ? -givens[start[l] + r] : givens[start[l] + r];
      const double co = std::cos(th), t = std::tan(th);
      if (!(std::abs(co) >= kGivens2MinCos)) return false;
      const int i = l % 2 + 2 * r;
      c.push_back(-t * a[i + 1] / a[i]);
      c.push_back(t * a[i] / a[i + 1]);
      a[i] *= co;
      a[i + 1] *= co;
    }
  }
  for (int i = 0; i < n; ++i) c.push_back(a[i] * gain);
  return true;
}

// Sub-block post-adjustment behind a deferred-scale DCT-2 (AxisOp::kDeferredSub): the k x k
// block acts on held values, so the scales of its k inputs are folded into its columns.
inline void fold_sub_scales(int n, int k, std::vector<double>& block) {
  for (int r = 0; r < k; ++r)
    for (int j = 0; j < k; ++j) block[r * k + j] *= deferred_scale_of<ST_DCT2>(n, j);
}

}  // namespace dctadj

/* dctadj_oracle.h -- CPU parity oracle (TEST INFRASTRUCTURE ONLY).
 * See dctadj_oracle.c for the reference file:line each function restates. */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_BASE_DCT2 = 0, OR_BASE_DST3 = 1, OR_BASE_DCT3 = 2 };
enum { OR_ADJ_NONE = 0, OR_ADJ_BAND = 1, OR_ADJ_SUBBLOCK = 2, OR_ADJ_DENSE = 3 };
enum { OR_SIDE_PRE = 0, OR_SIDE_POST = 1 };

/* one axis of an adjusted transform: base, adjustment kind/side, and the
 * realized N x N adjustment (row-major float64; unused when adj == NONE) */
typedef struct {
  int32_t n, base, adj, side, taps, order;
  const double* mat;
} or_axis;

int or_dct2(const double* x, double* y, int64_t nvec, int n);
int or_idct2(const double* x, double* y, int64_t nvec, int n);
int or_dst3(const double* x, double* y, int64_t nvec, int n);
int or_idst3(const double* x, double* y, int64_t nvec, int n);
int or_band(const double* a, int taps, const double* x, double* y, int64_t nvec, int n);
int or_subblock(const double* blk, int b, const double* x, double* y, int64_t nvec, int n);
int or_dense(const double* m, int rows, const double* x, double* y, int64_t nvec, int n);
int or_adjusted_1d(const or_axis* ax, int inverse, const double* x, double* y, int64_t nvec);
int or_adjusted_2d(const or_axis* ah, const or_axis* av, int inverse,
                   const double* x, double* y, int64_t nblk, int threads);
int or_adjusted_2d_f32(const or_axis* ah, const or_axis* av, int inverse,
                       const float* x, float* y, int64_t nblk, int threads);
int or_num_threads_available(void);

/* full-batch parity checkers (see dctadj_oracle.c); dtype 0 = fp32, 1 = fp64 */
typedef struct {
  double max_err; /* worst per-block normwise relative error */
  int64_t worst;  /* its block index (-1: no blocks) */
  int64_t over;   /* blocks with error > tol */
} or_check_result;
int or_check_2d(const or_axis* ah, const or_axis* av, int inverse, int dtype, const void* x,
                const void* y, int64_t nblk, int threads, double tol, or_check_result* res);
int or_check_mixed(const or_axis* table, int ntable, const int32_t* h_index,
                   const int32_t* v_index, const int64_t* offsets, int64_t nblk, int inverse,
                   int dtype, const void* x, const void* y, int threads, double tol,
                   or_check_result* res);
int or_check_frames(const or_axis* ah, const or_axis* av, int inverse, const float* frames,
                    const float* coefs, int nframes, int height, int width, int threads,
                    double tol, or_check_result* res);

#ifdef __cplusplus
}
#endif

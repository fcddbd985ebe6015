/*
 * dctadj.h -- C-ABI of the B200 adjusted-transform engine (libdctadj.so).
 *
 * Drop-in boundary for the reference's kernel plugin API
 * (reference pkg/src/dctadjust/kernels/__init__.py:33-41, a backend module
 * exporting dct2/idct2/dst3/idst3/band/subblock/dense over (nvec, N) batches)
 * and for its pipeline entry points forward_adjusted / inverse_adjusted
 * (reference pkg/src/dctadjust/pipeline.py:176-191).  The 2-D, frame and mixed
 * entries have no reference counterpart: they fuse the reference's 2-D
 * composition (rows then columns, pipeline.py:236-239) into one kernel.
 *
 * Conventions
 *  - Plain C types only.  `x`/`y` are DEVICE pointers (row-major, contiguous)
 *    unless the name ends in _host; `stream` is a cudaStream_t (NULL = legacy
 *    default stream).  Calls are stream-ordered, reentrant and never block the
 *    host, except the *_host entries, which return when the host output is
 *    written.
 *  - Adjustment matrices (`a`, `blk`, `m`, dctadj_axis.mat) are HOST float64
 *    arrays, read during the call (packed into the launch), never retained.
 *  - dtype: DCTADJ_F32 or DCTADJ_F64; inputs and outputs share it.
 *  - Outputs are caller-allocated and must not alias inputs.
 *  - Return value: DCTADJ_OK or an error code; no exception crosses the ABI.
 *    Codes map 1:1 onto the reference's error classes (errors.py:4-37):
 *    DIMENSION->InvalidDimensionError, SHAPE->ShapeError,
 *    PATTERN->PatternError, CONFIG->ConfigurationError,
 *    KIND->KindMismatchError, VALUE->ValueError.  dctadj_last_error() returns
 *    the calling thread's last message.
 */
#ifndef DCTADJ_H_
#define DCTADJ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum dctadj_status {
  DCTADJ_OK = 0,
  DCTADJ_ERR_DIMENSION = 1,   /* InvalidDimensionError (pipeline.py:40-44) */
  DCTADJ_ERR_SHAPE = 2,       /* ShapeError (pipeline.py:47-57) */
  DCTADJ_ERR_PATTERN = 3,     /* PatternError (pipeline.py:92-104) */
  DCTADJ_ERR_CONFIG = 4,      /* ConfigurationError (pipeline.py:141-148) */
  DCTADJ_ERR_KIND = 5,        /* KindMismatchError (errors.py:16-17) */
  DCTADJ_ERR_CUDA = 6,        /* CUDA runtime / driver failure */
  DCTADJ_ERR_UNSUPPORTED = 7, /* no kernel for this configuration */
  DCTADJ_ERR_VALUE = 8        /* ValueError (e.g. N > 64, _fastcore.pyx:194-195) */
};

enum dctadj_dtype { DCTADJ_F32 = 0, DCTADJ_F64 = 1 };

/* base transform of one axis (reference transforms.py TransformKind) */
enum dctadj_base {
  DCTADJ_BASE_DCT2 = 0, /* FAST_DCT2 (pipeline.py:35-37) */
  DCTADJ_BASE_DST3 = 1, /* FAST_DST3_VIA_DCT2 */
  DCTADJ_BASE_DCT3 = 2  /* DCT-3 = DCT-2^T: the DCT-8 pre flip */
};
/* adjustment pattern kind (reference design.py:43-46) and side (design.py:49-51) */
enum dctadj_adj { DCTADJ_ADJ_NONE = 0, DCTADJ_ADJ_BAND = 1, DCTADJ_ADJ_SUBBLOCK = 2,
                  DCTADJ_ADJ_DENSE = 3 };
enum dctadj_side { DCTADJ_SIDE_PRE = 0, DCTADJ_SIDE_POST = 1 };

/* One axis of an adjusted transform: the reference AdjustedTransform
 * (pipeline.py:127-135) flattened to plain data. */
typedef struct dctadj_axis {
  int32_t n;          /* transform length: 4, 8, 16, 32 or 64 (FAST_SIZES) */
  int32_t base;       /* dctadj_base */
  int32_t adj;        /* dctadj_adj */
  int32_t side;       /* dctadj_side */
  int32_t taps;       /* band taps (adj == BAND) */
  int32_t order;      /* sub-block order (adj == SUBBLOCK) */
  const double* mat;  /* host n x n realized adjustment (row-major); NULL if NONE */
  /* optional, band only: the Givens schedule behind `mat` -- taps-1 brick-wall
   * layers of adjacent-pair rotations (layer l pairs (i, i+1), i = l%2, l%2+2, ...;
   * reference design.py:225-243), angles in layer order, ascending i.  When given
   * (ngivens == the rotation count of that structure) the band runs as lifting
   * rotations (3 FMAs per rotation) instead of the 2*taps-1 FMA product. */
  const double* givens;
  int32_t ngivens;
  int32_t reserved;   /* 0 */
} dctadj_axis;

/* ---- the seven batch primitives (reference kernels/__init__.py:33-41) ----
 * x, y: (nvec, n) row-major device arrays. */
int dctadj_dct2(const void* x, void* y, int64_t nvec, int32_t n, int32_t dtype, void* stream);
int dctadj_idct2(const void* x, void* y, int64_t nvec, int32_t n, int32_t dtype, void* stream);
int dctadj_dst3(const void* x, void* y, int64_t nvec, int32_t n, int32_t dtype, void* stream);
int dctadj_idst3(const void* x, void* y, int64_t nvec, int32_t n, int32_t dtype, void* stream);
/* y[i,r] = sum_{|r-j|<taps} a[r,j] x[i,j]; a: host n x n  (_fastcore.pyx:253-273) */
int dctadj_band(const double* a, int32_t taps, const void* x, void* y, int64_t nvec, int32_t n,
                int32_t dtype, void* stream);
/* y = x with y[i,0:b] = blk x[i,0:b]; blk: host b x b; tail copied (_fastcore.pyx:276-290) */
int dctadj_subblock(const double* blk, int32_t b, const void* x, void* y, int64_t nvec,
                    int32_t n, int32_t dtype, void* stream);
/* y (nvec, rows) = x m^T; m: host rows x n  (_fastcore.pyx:293-307) */
int dctadj_dense(const double* m, int32_t rows, const void* x, void* y, int64_t nvec, int32_t n,
                 int32_t dtype, void* stream);

/* ---- fused 1-D adjusted transforms (pipeline.py:176-191) ---- */
int dctadj_forward_1d(const dctadj_axis* ax, const void* x, void* y, int64_t nvec, int32_t dtype,
                      void* stream);
int dctadj_inverse_1d(const dctadj_axis* ax, const void* y, void* x, int64_t nvec, int32_t dtype,
                      void* stream);

/* ---- fused 2-D separable transforms over (nblk, H, W) blocks ----
 * h: row axis (length W), v: column axis (length H).
 * forward: Y = T_v X T_h^T (rows, then columns); inverse: X = T_v^T Y T_h. */
int dctadj_forward_2d(const dctadj_axis* h, const dctadj_axis* v, const void* x, void* y,
                      int64_t nblk, int32_t dtype, void* stream);
int dctadj_inverse_2d(const dctadj_axis* h, const dctadj_axis* v, const void* y, void* x,
                      int64_t nblk, int32_t dtype, void* stream);
/* Round trip (config 2's step): y = forward(x) and xr = inverse(y) in one
 * pass over HBM (x read once, y and xr written once: 12 B per coefficient pair
 * in fp32 instead of 16 B).  Results are bit-identical to dctadj_forward_2d
 * followed by dctadj_inverse_2d; op pairs without a fused kernel run as exactly
 * those two calls.  xr may alias x; y must not alias xr.  Composes the
 * reference's forward_adjusted / inverse_adjusted (pipeline.py:176-191). */
int dctadj_roundtrip_2d(const dctadj_axis* h, const dctadj_axis* v, const void* x, void* y,
                        void* xr, int64_t nblk, int32_t dtype, void* stream);
/* 1 when dctadj_roundtrip_2d runs these axes / dtype as the fused kernel, 0
 * when it runs the two separate kernels (or the arguments are invalid). */
int dctadj_roundtrip_fused(const dctadj_axis* h, const dctadj_axis* v, int32_t dtype);

/* Host-buffer variants: x_host/y_host are host arrays (pinned for full speed);
 * copies, kernels and read-back are pipelined over chunks on internal streams.
 * Blocks until y_host is written.  device: CUDA ordinal to run on. */
int dctadj_forward_2d_host(const dctadj_axis* h, const dctadj_axis* v, const void* x_host,
                           void* y_host, int64_t nblk, int32_t dtype, int32_t device);
int dctadj_inverse_2d_host(const dctadj_axis* h, const dctadj_axis* v, const void* y_host,
                           void* x_host, int64_t nblk, int32_t dtype, int32_t device);
/* Round trip on host buffers (config 2's step): y_host = forward(x_host) and
 * xr_host = inverse(y_host), the inverse run on the device-resident
 * coefficients of each chunk (one H2D, two D2H per chunk).  Same results as
 * dctadj_forward_2d_host followed by dctadj_inverse_2d_host.  Composes the
 * reference's forward_adjusted / inverse_adjusted (pipeline.py:176-191). */
int dctadj_roundtrip_2d_host(const dctadj_axis* h, const dctadj_axis* v, const void* x_host,
                             void* y_host, void* xr_host, int64_t nblk, int32_t dtype,
                             int32_t device);

/* ---- frame tiling: frames (nframes, height, width) <-> block-major
 * coefficients (nframes * ceil(height/H) * (width/W), H, W).  Rows past
 * `height` are zero padding on the way in and clipped on the way out. */
int dctadj_forward_frames(const dctadj_axis* h, const dctadj_axis* v, const void* frames,
                          void* coefs, int32_t nframes, int32_t height, int32_t width,
                          int32_t dtype, void* stream);
int dctadj_inverse_frames(const dctadj_axis* h, const dctadj_axis* v, const void* coefs,
                          void* frames, int32_t nframes, int32_t height, int32_t width,
                          int32_t dtype, void* stream);

/* Config 5's comparison step in one call: the adjusted forward (h, v) AND the
 * exact forward (eh, ev; typically dense DST-7) of the same frames, plus the
 * per-frame approximation error err[f*4 + {0,1,2,3}] = {sum (Ya - Ye)^2,
 * sum Ye^2} over all tiles and over tile rows entirely inside `height` (err may
 * be NULL; it is zeroed first).  fp32 32x32 with a sub-block-8 post or band-6
 * (Givens) pre adjustment on both axes, dense exact axes and width a multiple of
 * 128 runs as ONE tensor-core kernel that reads the frames once
 * (csrc/dense_tc.cuh, FUSED); anything else runs the two frame transforms and a
 * reduction.  The error sums are defined on 32x32 tiles: other block sizes
 * with err != NULL return DCTADJ_ERR_UNSUPPORTED (with err = NULL they run).  Replaces the reference's two transform calls plus its error sum
 * (reference pipeline.py:176-199). */
int dctadj_forward_frames_exact(const dctadj_axis* h, const dctadj_axis* v, const dctadj_axis* eh,
                                const dctadj_axis* ev, const void* frames, void* coefs,
                                void* exact, double* err, int32_t nframes, int32_t height,
                                int32_t width, int32_t dtype, void* stream);

/* ---- simultaneous encoder evaluation (reference pipeline.py:256-293, paper
 * Table 1 "Multiple"): for each (H, W) block, one read, one shared 2-D DCT-2 and
 * five coefficient planes, planes[k] (device, each (nblk, H, W)):
 *   0 (dct2, dct2)  1 (dst7, dst7)  2 (dct8, dst7)  3 (dst7, dct8)  4 (dct8, dct8)
 * keyed (horizontal, vertical).  h / v: post sub-block DCT-2 -> DST-7 axes (the
 * DCT-8 planes use C8 = S C7 S, design.py:677-715).  Coefficients outside the
 * leading 8 rows / columns are bit-identical across all five planes. */
int dctadj_encoder_eval(const dctadj_axis* h, const dctadj_axis* v, const void* x,
                        void* const* planes, int64_t nblk, int32_t dtype, void* stream);

/* ---- mixed-shape batches (config 3): blocks of different sizes packed back
 * to back in one buffer of `total_elements` samples.  Block i starts at element
 * offsets[i] (a multiple of its width), its rows use axis-table entry
 * h_index[i] (width = sizes[h_index[i]]) and its columns entry v_index[i]
 * (height = sizes[v_index[i]]).  The plan buckets blocks by (h, v) class once
 * (host arrays in, device offset lists kept); each call then runs one gather
 * kernel per class.  `table` (ntable entries, sizes as in the plan) is read per
 * call, so the same plan serves pre- and post-adjusted runs. */
typedef struct dctadj_mixed dctadj_mixed;
int dctadj_mixed_create(const int64_t* offsets, const int32_t* h_index, const int32_t* v_index,
                        int64_t nblk, const int32_t* sizes, int32_t ntable,
                        int64_t total_elements, dctadj_mixed** plan);
int dctadj_mixed_forward(const dctadj_mixed* plan, const dctadj_axis* table, const void* x,
                         void* y, int32_t dtype, void* stream);
int dctadj_mixed_inverse(const dctadj_mixed* plan, const dctadj_axis* table, const void* y,
                         void* x, int32_t dtype, void* stream);
/* forward then inverse of the whole mixed batch (y = forward(x), xr =
 * inverse(y)) with one fused gather kernel per class (x read once, y and xr
 * written once); bit-identical to dctadj_mixed_forward + dctadj_mixed_inverse,
 * which it runs when a class has no fused kernel.  y must not alias xr. */
int dctadj_mixed_roundtrip(const dctadj_mixed* plan, const dctadj_axis* table, const void* x,
                           void* y, void* xr, int32_t dtype, void* stream);
/* 1 when dctadj_mixed_roundtrip runs this plan / table / dtype as fused kernels */
int dctadj_mixed_roundtrip_fused(const dctadj_mixed* plan, const dctadj_axis* table,
                                 int32_t dtype);
int dctadj_mixed_destroy(dctadj_mixed* plan);

/* ---- diagnostics ---- */
/* The tile pipeline with no arithmetic (TMA load -> smem -> TMA store) on
 * (nblk, h, w) blocks, h x w in {32x32, 64x64, 16x16}: the data-movement
 * ceiling the transform kernels are measured against. */
int dctadj_copy_tiles(const void* x, void* y, int64_t nblk, int32_t h, int32_t w, int32_t dtype,
                      void* stream);
const char* dctadj_status_string(int32_t status);
const char* dctadj_last_error(void);
int32_t dctadj_version(void);
/* number of tile_kernel instantiations compiled into this library */
int32_t dctadj_kernel_count(void);
/* the device cache of dense matrices (composites, exact comparison transforms):
 * entries held and entries pinned by calls still in flight (0 between calls) */
int dctadj_dense_cache_state(int32_t* entries, int32_t* pinned);
/* The cross-launch overlap rule, as the launchers apply it (no device work):
 * would a launch on `stream` reading [in, in + in_bytes) and writing
 * [out, out + out_bytes) skip its entry wait on the previous grid -- 1 yes, 0 no
 * -- given every launch recorded there since the last one that waited?  The
 * probe is recorded like a launch.  poison != 0 instead records a launch whose
 * ranges are unknown (the next launch waits).  Returns 0 / 1, or < 0 on error. */
int dctadj_pdl_probe(void* stream, const void* in, uint64_t in_bytes, const void* out,
                     uint64_t out_bytes, int32_t poison);
/* 1 when the library was built with DCTADJ_TUNING=1 (measured-slower tuning
 * variants selectable by DCTADJ_VARIANT / DCTADJ_RT_VARIANT), else 0 */
int32_t dctadj_tuning_build(void);

/* ---- adjustment designer (offline) ----
 * The reference's cyclic coordinate descent over the angles of a rotation
 * skeleton (design.py:377-543, the optimize_adjustment path without the
 * sparsity penalty), every restart in its own CTA.  Host arrays in / out:
 * base, desired: n x n row-major (n <= 64); weights: n; side 0 = pre
 * (H = B A), 1 = post (H = A B); rotation t acts on (rp[t], rq[t]);
 * theta0: restarts x m start angles.  Out: theta (restarts x m), trace
 * (restarts x (max_sweeps + 1) objectives; entry k after sweep k), sweeps
 * (trace length - 1) and converged flags per restart.  Blocks until done. */
int dctadj_design_cd(int32_t n, const double* base, const double* desired,
                     const double* weights, int32_t side, int32_t m, const int32_t* rp,
                     const int32_t* rq, int32_t restarts, const double* theta0,
                     int32_t max_sweeps, double tol, double* theta_out, double* trace_out,
                     int32_t* sweeps_out, int32_t* converged_out, int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* DCTADJ_H_ */

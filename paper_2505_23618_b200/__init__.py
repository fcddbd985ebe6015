"""B200-native adjusted DST-7 / DCT-8 transforms (arxiv 2505.23618).

A fast DCT-2-family butterfly plus a sparse orthogonal adjustment (band
pre-adjustment or 8x8 low-frequency post-adjustment), batched over residual
blocks, in hand-written sm_100a CUDA behind a C-ABI (include/dctadj.h).
The Python surface mirrors the reference package `dctadjust`:

  kernels   the 7-function plugin API (dct2, idct2, dst3, idst3, band, subblock, dense)
  pipeline  forward_adjusted / inverse_adjusted / make_adjusted_transform / fast_* /
            apply_band / apply_subblock / dense_matrix, plus the fused
            forward_adjusted_2d / inverse_adjusted_2d / forward_frames / inverse_frames
  design    adjustment records (AdjustmentMatrix, SparsityPattern, GivensSchedule, ...)
  matio     the reference's adjustment / matrix text formats; shipped designs
  transforms exact matrices (comparison paths)
"""
from .errors import (ConfigurationError, CudaError, DctAdjustError, InvalidDimensionError,
                     InvalidScheduleError, KindMismatchError, MatrixFormatError, PatternError,
                     ShapeError, UnsupportedError)
from .transforms import TransformKind, build_transform, alternating_signs, flip_to_dct8
from .design import (AdjustmentMatrix, GivensSchedule, PatternKind, PlaneRotation, Side,
                     SparsityPattern, dct8_adjustment_from_dst7, flip_pre_adjustment,
                     givens_to_matrix, identity_adjustment, pattern_schedule_template,
                     random_adjustment)

__version__ = "0.1.0"
KERNEL_BACKEND = "cuda"

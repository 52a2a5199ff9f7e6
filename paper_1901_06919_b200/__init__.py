"""B200-native Fourier Disparity Layers: the construction and rendering hot paths.

Drop-in for the reference package `fdl` on these paths (same names, argument
meaning and exceptions as fdl/__init__.py:3-98 for everything below); the
compute runs in hand-written sm_100a CUDA kernels behind a C ABI
(include/fdl_b200.h, libfdl_b200.so).  FDL1 model files are read and
written straight from / into device memory (io.py);
calibration runs its batch solves, objective and gradients on the GPU
(calibrate.py), and so do the interpolate / denoise
pipelines built on it (pipeline.py, row 2).
Out of scope: CLI, HTTP service, viewer.
"""

from .spectra import DFT_CONVENTION, FrequencyGrid
from .lfmodel import GAMMA, LINEAR, ApertureSpec, FdlModel, QuantisedImages, ShiftParams, ViewSet, expand_shifts
from .construct import (
    DEFAULT_EPS,
    SOLVE_CHUNK,
    RankDeficiencyError,
    build_system_row,
    construct_fdl,
    solve_frequency,
    default_lambda,
    last_construct_stats,
    view_regularizer,
)
from .render import (
    RenderRequest,
    RenderStats,
    aperture_spectrum,
    last_render_stats,
    render,
    render_many,
    render_views_with_shifts,
    srgb_decode,
    srgb_encode,
)

from .io import ModelFormatError, load_model, save_model
from .calibrate import (
    CalibConfig,
    CalibrationDivergence,
    CalibrationResult,
    calibrate,
    calibrate_relaxed,
    grad_factored,
    grad_shift_matrix,
    layer_coefficients,
    layer_regularizer,
    objective,
    regauge_to_coords,
)
from .pipeline import PipelineConfig, QualityReport, denoise, interpolate_views, psnr

__version__ = "0.1.0"

__all__ = [
    "PipelineConfig",
    "QualityReport",
    "denoise",
    "interpolate_views",
    "psnr",
    "CalibConfig",
    "CalibrationDivergence",
    "CalibrationResult",
    "calibrate",
    "calibrate_relaxed",
    "grad_factored",
    "grad_shift_matrix",
    "layer_coefficients",
    "layer_regularizer",
    "objective",
    "regauge_to_coords",
    "DFT_CONVENTION",
    "FrequencyGrid",
    "GAMMA",
    "LINEAR",
    "ApertureSpec",
    "FdlModel",
    "ShiftParams",
    "QuantisedImages",
    "ViewSet",
    "expand_shifts",
    "DEFAULT_EPS",
    "SOLVE_CHUNK",
    "RankDeficiencyError",
    "build_system_row",
    "construct_fdl",
    "solve_frequency",
    "default_lambda",
    "last_construct_stats",
    "view_regularizer",
    "RenderRequest",
    "RenderStats",
    "aperture_spectrum",
    "last_render_stats",
    "render",
    "render_many",
    "render_views_with_shifts",
    "srgb_decode",
    "srgb_encode",
    "ModelFormatError",
    "load_model",
    "save_model",
    "__version__",
]

"""ctypes binding of libfdl_b200.so (include/fdl_b200.h).

The product path has no CPU fallback: if the library is missing or there is no
CUDA device, every hot-path call raises.  PyTorch is only the memory/stream
plumbing here: buffers are torch CUDA tensors whose raw pointers go through
the C ABI together with torch's current stream.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libfdl_b200.so"

FDL_OK = 0
FDL_BIN_SUSPECT = 2
FDL_ERR_INVALID = -1
FDL_ERR_CUDA = -2
FDL_ERR_UNSUPPORTED = -3
FDL_ERR_RANK = -4


class FdlNativeError(RuntimeError):
    """A CUDA / cuFFT / unsupported-shape failure inside libfdl_b200."""


c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_double_p = ctypes.POINTER(ctypes.c_double)


class FdlAperture(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
        ("table_re", c_double_p), ("table_im", c_double_p),
        ("xi0_x", ctypes.c_double), ("step_x", ctypes.c_double),
        ("xi0_y", ctypes.c_double), ("step_y", ctypes.c_double),
    ]


class FdlSolveDesc(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int32), ("n", ctypes.c_int32), ("C", ctypes.c_int32),
        ("Hp", ctypes.c_int32), ("Wp", ctypes.c_int32),
        ("nrows", ctypes.c_int32), ("rows", c_int32_p),
        ("u", c_double_p), ("v", c_double_p), ("pu", c_double_p), ("pv", c_double_p),
        ("d", c_double_p),
        ("view_aperture", c_int32_p), ("s", c_double_p), ("scale", c_double_p),
        ("n_apertures", ctypes.c_int32), ("apertures", ctypes.POINTER(FdlAperture)),
        ("lam", ctypes.c_double), ("eps", ctypes.c_double),
        ("spectra_dev", ctypes.c_void_p), ("layers_dev", ctypes.c_void_p),
        ("status_dev", ctypes.c_void_p), ("force_path", ctypes.c_int32),
        ("plane_rows", ctypes.c_int32), ("lam_dev", ctypes.c_void_p),
    ]


class FdlRenderDesc(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("C", ctypes.c_int32), ("Hp", ctypes.c_int32), ("Wp", ctypes.c_int32),
        ("V", ctypes.c_int32),
        ("d", c_double_p), ("pu", c_double_p), ("pv", c_double_p), ("t", c_double_p),
        ("view_aperture", c_int32_p), ("n_apertures", ctypes.c_int32),
        ("apertures", ctypes.POINTER(FdlAperture)),
        ("layers_dev", ctypes.c_void_p), ("out_dev", ctypes.c_void_p), ("oob_dev", ctypes.c_void_p),
    ]


class FdlDenseDesc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32), ("m", ctypes.c_int32), ("n", ctypes.c_int32), ("C", ctypes.c_int32),
        ("A_dev", ctypes.c_void_p), ("b_dev", ctypes.c_void_p), ("reg_dev", ctypes.c_void_p),
        ("R_dev", ctypes.c_void_p), ("lam", ctypes.c_double), ("x_dev", ctypes.c_void_p),
        ("status_dev", ctypes.c_void_p),
    ]


class FdlCalibDesc(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int32), ("n", ctypes.c_int32), ("B", ctypes.c_int32),
        ("H", ctypes.c_int32), ("W", ctypes.c_int32),
        ("bins", c_int32_p), ("pu", c_double_p), ("pv", c_double_p), ("gamma", c_double_p),
        ("lam", ctypes.c_double),
        ("spec_dev", ctypes.c_void_p), ("x_dev", ctypes.c_void_p), ("status_dev", ctypes.c_void_p),
        ("gfall_dev", ctypes.c_void_p), ("rfall_dev", ctypes.c_void_p),
        ("obj_dev", ctypes.c_void_p), ("grad_dev", ctypes.c_void_p),
    ]


_lock = threading.Lock()
_lib = None

EXPORTS = {
    "fdl_version": (ctypes.c_int, []),
    "fdl_last_error": (ctypes.c_char_p, []),
    "fdl_selftest": (ctypes.c_int, [c_double_p]),
    "fdl_kernel_timer": (ctypes.c_int, [ctypes.c_int32]),
    "fdl_kernel_timer_read": (ctypes.c_int, [ctypes.c_int32, c_double_p, c_int32_p]),
    "fdl_fft_force_cufft": (ctypes.c_int, [ctypes.c_int32]),
    "fdl_staging_arena_begin": (ctypes.c_void_p, []),
    "fdl_staging_arena_end": (ctypes.c_int, [ctypes.c_void_p]),
    "fdl_staging_arena_free": (ctypes.c_int, [ctypes.c_void_p]),
    "fdl_default_lambda": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "fdl_views_to_spectra_workspace": (ctypes.c_size_t, [ctypes.c_int32] * 5),
    "fdl_views_to_spectra": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int32] * 5 + [
        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "fdl_views_to_spectra_srgb": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int32] * 5 + [
        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "fdl_gather_rows": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int32] * 4 + [
        ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "fdl_solve_bins_workspace": (ctypes.c_size_t, [ctypes.POINTER(FdlSolveDesc)]),
    "fdl_solve_bins": (ctypes.c_int, [ctypes.POINTER(FdlSolveDesc), ctypes.c_void_p, ctypes.c_size_t,
                                      c_int32_p, ctypes.c_void_p]),
    "fdl_solve_path": (ctypes.c_int, [ctypes.POINTER(FdlSolveDesc)]),
    "fdl_resolve_bins_workspace": (ctypes.c_size_t, [ctypes.POINTER(FdlSolveDesc), ctypes.c_int32]),
    "fdl_resolve_bins": (ctypes.c_int, [ctypes.POINTER(FdlSolveDesc), c_int32_p, ctypes.c_int32, ctypes.c_void_p,
                                        ctypes.c_size_t, ctypes.c_void_p]),
    "fdl_audit_bins": (ctypes.c_int, [ctypes.POINTER(FdlSolveDesc), c_int32_p, ctypes.c_int32, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "fdl_solve_dense_workspace": (ctypes.c_size_t, [ctypes.POINTER(FdlDenseDesc)]),
    "fdl_solve_dense": (ctypes.c_int, [ctypes.POINTER(FdlDenseDesc), ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p]),
    "fdl_lstsq_minnorm_workspace": (ctypes.c_size_t, [ctypes.c_int32] * 4),
    "fdl_lstsq_minnorm": (ctypes.c_int, [ctypes.c_int32] * 4 + [ctypes.c_void_p] * 4 + [
        ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "fdl_calib_workspace": (ctypes.c_size_t, [ctypes.POINTER(FdlCalibDesc)]),
    "fdl_calib_solve": (ctypes.c_int, [ctypes.POINTER(FdlCalibDesc), ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p]),
    "fdl_calib_terms": (ctypes.c_int, [ctypes.POINTER(FdlCalibDesc), ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p]),
    "fdl_symmetrize": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int32] * 5 + [
        c_int32_p, c_int32_p, ctypes.c_void_p]),
    "fdl_symmetrize_rows": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int32] * 5 + [c_int32_p, ctypes.c_void_p]),
    "fdl_rows_to_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int32] * 5 + [ctypes.c_void_p]),
    "fdl_render_workspace": (ctypes.c_size_t, [ctypes.POINTER(FdlRenderDesc)]),
    "fdl_render_workspace_bound": (ctypes.c_size_t, [ctypes.c_int32] * 6 + [ctypes.c_int64]),
    "fdl_render_spectra": (ctypes.c_int, [ctypes.POINTER(FdlRenderDesc), ctypes.c_void_p,
                                          ctypes.c_size_t, ctypes.c_void_p]),
    "fdl_view_sqerr_workspace": (ctypes.c_size_t, [ctypes.c_int32] * 2),
    "fdl_view_sqerr": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int32] * 5 + [
        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "fdl_images_to_u8": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "fdl_dequantise_views": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p,
                                            ctypes.c_void_p]),
    "fdl_spectra_to_images_workspace": (ctypes.c_size_t, [ctypes.c_int32] * 4),
    "fdl_spectra_to_images": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int32] * 8 + [
        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
}


def lib():
    """The loaded library (raises ImportError when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1901_06919_b200.build_native` "
                    "(there is no CPU fallback)")
            handle = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in EXPORTS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(rc: int, what: str):
    if rc == FDL_OK:
        return
    msg = lib().fdl_last_error().decode(errors="replace")
    if rc == FDL_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    if rc == FDL_ERR_RANK:
        from .construct import RankDeficiencyError
        raise RankDeficiencyError(f"{what}: {msg}")
    raise FdlNativeError(f"{what} failed ({rc}): {msg}")


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

def dptr(arr) -> c_double_p:
    """Pointer into a C-contiguous float64 numpy array (caller keeps it alive)."""
    if arr is None:
        return None
    assert arr.dtype == np.float64 and arr.flags.c_contiguous
    return arr.ctypes.data_as(c_double_p)


def iptr(arr) -> c_int32_p:
    if arr is None:
        return None
    assert arr.dtype == np.int32 and arr.flags.c_contiguous
    return arr.ctypes.data_as(c_int32_p)


def aperture_structs(specs):
    """(ctypes array of FdlAperture, keepalive list) for a list of ApertureSpec."""
    keep = []
    arr = (FdlAperture * max(len(specs), 1))()
    for i, ap in enumerate(specs):
        table = np.asarray(ap.table)
        re = np.ascontiguousarray(table.real, dtype=np.float64)
        im = np.ascontiguousarray(table.imag, dtype=np.float64) if np.iscomplexobj(table) else None
        keep += [re, im]
        xi_x = np.asarray(ap.xi_x, dtype=np.float64)
        xi_y = np.asarray(ap.xi_y, dtype=np.float64)
        arr[i] = FdlAperture(rows=table.shape[0], cols=table.shape[1], table_re=dptr(re),
                             table_im=dptr(im) if im is not None else None,
                             # lfmodel.py:73-74: step = axis[1] - axis[0], pos from axis[0]
                             xi0_x=float(xi_x[0]), step_x=float(xi_x[1] - xi_x[0]),
                             xi0_y=float(xi_y[0]), step_y=float(xi_y[1] - xi_y[0]))
    return arr, keep


def on_device(pick):
    """Decorator: run the call with the CUDA device `pick(*args, **kwargs)` current
    (None: leave the current device).  The native layer launches on the
    current device's streams and keeps per-device staging, so every host entry
    point selects the device of the tensors it is handed first."""
    import functools

    def deco(fn):
        @functools.wraps(fn)
        def call(*args, **kwargs):
            dev = pick(*args, **kwargs)
            if dev is None:
                return fn(*args, **kwargs)
            import torch
            dev = torch.device(dev)
            if dev.type != "cuda":
                return fn(*args, **kwargs)
            with torch.cuda.device(dev):
                return fn(*args, **kwargs)
        return call
    return deco


def stream_handle(device=None):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def workspace(nbytes: int, device):
    import torch
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


_copy_streams = threading.local()


def copy_stream(device):
    """A per-thread, per-device side stream for host<->device copies that overlap
    the kernels on the current stream."""
    import torch
    cache = getattr(_copy_streams, "by_dev", None)
    if cache is None:
        cache = _copy_streams.by_dev = {}
    key = torch.device(device).index
    s = cache.get(key)
    if s is None:
        s = cache[key] = torch.cuda.Stream(device=device)
    return s

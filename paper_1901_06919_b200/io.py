"""FDL1 model files straight from / into device memory (reference: fdl/io.py:157-237).

The on-disk payload is the layers as complex64 in (n, C, Hp, Whp) order --
exactly the layout K1 writes in HBM -- so `save_model` copies the device
tensor once into pinned host memory (or reuses the overlapped read-back that
`construct_fdl` already made, `FdlModel.layers_host()`) and writes it without
the reference's complex128 round trip, and `load_model` reads the payload
into pinned memory and uploads it once: the returned model's layers live on
the GPU (`layers_device()`), `.layers` stays the reference's complex128 view.

File layout (io.py:34-35, 157-180), little-endian:
    header  <4sIIIIIBB16sId : magic b"FDL1", width, height, pad_margin, n,
            channels, linear flag, calibration kind (0 none, 1 factored,
            2 relaxed), DFT convention (16 bytes, NUL padded), views m,
            lambda (NaN = none)
    d       n float64
    layers  n*C*Hp*Whp complex64
    kind 1: u (m float64), v (m float64); kind 2: pu (m*n), pv (m*n) float64

Errors follow the reference: ModelFormatError (a ValueError) for a short
file, bad magic, unknown convention or calibration kind, and a payload
whose size disagrees with the header.
"""

from __future__ import annotations

import math
import struct
from pathlib import Path

import numpy as np

from .lfmodel import GAMMA, LINEAR, FdlModel, ShiftParams
from .spectra import DFT_CONVENTION, FrequencyGrid

__all__ = ["MAGIC", "ModelFormatError", "save_model", "load_model"]

MAGIC = b"FDL1"
_HEADER = struct.Struct("<4sIIIIIBB16sId")  # io.py:35


class ModelFormatError(ValueError):
    """Malformed FDL1 model file (io.py:42-43)."""


def _layers_c64_bytes(model: FdlModel) -> memoryview:
    """The layers as contiguous complex64 bytes, from device memory when the
    model lives there (one pinned D2H copy, or the construction's read-back)."""
    if model._host is None or model._dev is not None or model._host_async is not None:
        t = model.layers_host()  # pinned complex64 (n, C, Hp, Whp)
        return memoryview(t.contiguous().numpy()).cast("B")
    return memoryview(np.ascontiguousarray(model._host.astype(np.complex64))).cast("B")


def save_model(path, model: FdlModel) -> None:
    """Serialize an FdlModel to the FDL1 binary format (io.py:157-180)."""
    calib = model.calibration
    if calib is None:
        kind, m = 0, 0
    elif calib.is_factored:
        kind, m = 1, calib.num_views
    else:
        kind, m = 2, calib.num_views
    lam = model.lambda_used if model.lambda_used is not None else math.nan
    header = _HEADER.pack(
        MAGIC, model.width, model.height, model.pad_margin, model.num_layers,
        model.channels, 1 if model.color_space == LINEAR else 0, kind,
        model.convention.encode()[:16].ljust(16, b"\0"), m, lam,
    )
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(np.ascontiguousarray(model.disparities, dtype="<f8").tobytes())
        fh.write(_layers_c64_bytes(model))
        if kind == 1:
            fh.write(np.ascontiguousarray(calib.u, dtype="<f8").tobytes())
            fh.write(np.ascontiguousarray(calib.v, dtype="<f8").tobytes())
        elif kind == 2:
            fh.write(np.ascontiguousarray(calib.pu, dtype="<f8").tobytes())
            fh.write(np.ascontiguousarray(calib.pv, dtype="<f8").tobytes())


def load_model(path, device=None) -> FdlModel:
    """Read an FDL1 model file (io.py:183-237); rejects bad magic and
    truncated payloads.  With CUDA available the layers are uploaded once to
    `device` (default: the current device) as complex64."""
    raw = Path(path).read_bytes()
    if len(raw) < _HEADER.size:
        raise ModelFormatError(f"file too small for a model header: {path}")
    magic, w, h, pad, n, c, gamma_flag, kind, conv, m, lam = _HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise ModelFormatError(f"bad magic {magic!r}; not an FDL1 model file")
    convention = conv.rstrip(b"\0").decode()
    if convention != DFT_CONVENTION:
        raise ModelFormatError(f"unsupported transform convention {convention!r}")
    hp, wp = h + 2 * pad, w + 2 * pad
    whp = wp // 2 + 1
    sizes = [n * 8, n * c * hp * whp * 8]
    if kind == 1:
        sizes += [m * 8, m * 8]
    elif kind == 2:
        sizes += [m * n * 8, m * n * 8]
    elif kind != 0:
        raise ModelFormatError(f"unknown calibration block kind {kind}")
    expected = _HEADER.size + sum(sizes)
    if len(raw) != expected:
        raise ModelFormatError(
            f"payload size mismatch: header implies {expected} bytes, file has {len(raw)}"
        )
    off = _HEADER.size
    d = np.frombuffer(raw, dtype="<f8", count=n, offset=off).copy()
    off += n * 8
    payload = np.frombuffer(raw, dtype=np.complex64, count=n * c * hp * whp, offset=off).reshape(n, c, hp, whp)
    off += n * c * hp * whp * 8
    layers = _upload(payload, device)
    calibration = None
    if kind == 1:
        u = np.frombuffer(raw, dtype="<f8", count=m, offset=off).copy()
        off += m * 8
        v = np.frombuffer(raw, dtype="<f8", count=m, offset=off).copy()
        calibration = ShiftParams.factored(u, v, d)
    elif kind == 2:
        pu = np.frombuffer(raw, dtype="<f8", count=m * n, offset=off).reshape(m, n).copy()
        off += m * n * 8
        pv = np.frombuffer(raw, dtype="<f8", count=m * n, offset=off).reshape(m, n).copy()
        calibration = ShiftParams.relaxed(pu, pv, d=d)
    return FdlModel(
        disparities=d,
        layers=layers,
        grid=FrequencyGrid(width=wp, height=hp),
        width=w,
        height=h,
        pad_margin=pad,
        color_space=LINEAR if gamma_flag else GAMMA,
        calibration=calibration,
        lambda_used=None if math.isnan(lam) else lam,
        convention=convention,
    )


def _upload(payload: np.ndarray, device):
    """complex64 payload -> CUDA tensor through one pinned staging copy; the
    reference's complex128 host array when there is no GPU (I/O is not a
    compute path: the render/construct kernels still require the device)."""
    try:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError
    except Exception:
        return payload.astype(np.complex128)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    host = torch.empty(payload.shape, dtype=torch.complex64, pin_memory=True)
    host.numpy()[...] = payload
    out = torch.empty(payload.shape, dtype=torch.complex64, device=dev)
    out.copy_(host, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()  # the pinned buffer is released on return
    return out

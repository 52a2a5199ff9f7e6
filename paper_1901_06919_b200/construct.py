"""FDL construction on the B200 (reference: fdl/construct.py:219-308).

`construct_fdl` keeps the reference signature, defaults and exceptions; the
work runs as three native stages through the C ABI (include/fdl_b200.h):

  K0 fdl_views_to_spectra  pad + cuFFT R2C + per-view sum |b|^2  (construct.py:250-266)
  K1 fdl_solve_bins        per-bin fp64 regularised LS            (construct.py:68-80,168-211)
  K2 fdl_symmetrize        self-conjugate column post-pass        (construct.py:286-297)

The default lambda (construct.py:214-216) is 1e-4 * sum|b|^2 / (Q m), with the
per-view partial sums added in view order so the value does not depend on how
the views are sharded across GPUs.
"""

from __future__ import annotations

import math
import os

import numpy as np

from . import _native as nat
from .lfmodel import GAMMA, LINEAR, FdlModel, QuantisedImages, ShiftParams, ViewSet, _is_torch
from .spectra import FrequencyGrid

__all__ = [
    "RankDeficiencyError",
    "build_system_row",
    "solve_frequency",
    "solve_dense",
    "DEFAULT_EPS",
    "SOLVE_CHUNK",
    "view_regularizer",
    "default_lambda",
    "construct_fdl",
    "ConstructStats",
    "last_construct_stats",
]

DEFAULT_EPS = 1e-9       # construct.py:27
SOLVE_CHUNK = 16384      # construct.py:28 (K1 solves every bin at once; the chunk is the fallback granularity)


class RankDeficiencyError(Exception):
    """Unregularized normal matrix is singular at some frequency (construct.py:32-33)."""


def view_regularizer(omega_x, omega_y, d, eps: float = DEFAULT_EPS):
    """Diagonal (wx^2+wy^2)^2 d_k^4 + eps of the view regulariser (construct.py:36-45)."""
    w4 = (np.asarray(omega_x, float) ** 2 + np.asarray(omega_y, float) ** 2) ** 2
    return w4[..., None] * np.asarray(d, float) ** 4 + eps


def build_system_row(view: ViewSet, j: int, omega, d, grid: FrequencyGrid | None = None):
    """System-matrix row of view j at frequency (wx, wy) (construct.py:83-109).

    A host helper (one row, n entries) with the reference's Nyquist handling;
    the construction itself generates A on the device.
    """
    wx, wy = float(omega[0]), float(omega[1])
    d = np.asarray(d, dtype=np.float64)
    pu, pv = view.u[j] * d, view.v[j] * d
    phx = np.exp(2j * np.pi * pu * wx)
    phy = np.exp(2j * np.pi * pv * wy)
    if grid is not None:
        if grid.width % 2 == 0 and wx == grid.omega_x[grid.width // 2]:
            phx = np.cos(np.pi * pu).astype(np.complex128)
        if grid.height % 2 == 0 and wy == grid.omega_y[grid.height // 2]:
            phy = np.cos(np.pi * pv).astype(np.complex128)
    row = phx * phy
    ap = view.apertures[j]
    if ap is not None and not ap.is_pinhole:
        t = view.aperture_scale[j] * (view.s[j] - d)
        row = row * ap.evaluate(t * wx, t * wy)
    return row


@nat.on_device(lambda A, b, reg, lam, device=None: device)
def solve_dense(A, b, reg, lam: float, device=None):
    """Batched explicit regularised solves on the GPU (fdl_solve_dense).

    A (B, m, n), b (B, m, C), reg (B, n) diagonal or (B, n, n) Hermitian.
    Returns (x (B, n, C) complex128 numpy, status (B,) int8): 0 normal
    equations accepted, 2 minimum-norm fallback used, 1 failed, 3 singular at lam = 0.
    """
    torch = _require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    A = np.ascontiguousarray(A, dtype=np.complex128)
    b = np.ascontiguousarray(b, dtype=np.complex128)
    B, m, n = A.shape
    C = b.shape[2]
    reg = np.asarray(reg)
    At = torch.from_numpy(A).to(dev)
    bt = torch.from_numpy(b).to(dev)
    x = torch.empty((B, n, C), dtype=torch.complex128, device=dev)
    status = torch.zeros(B, dtype=torch.int8, device=dev)
    desc = nat.FdlDenseDesc()
    desc.batch, desc.m, desc.n, desc.C = B, m, n, C
    desc.A_dev, desc.b_dev, desc.x_dev, desc.status_dev = At.data_ptr(), bt.data_ptr(), x.data_ptr(), status.data_ptr()
    keep = []
    if reg.ndim == 2 and reg.shape == (B, n):
        rt = torch.from_numpy(np.ascontiguousarray(reg, dtype=np.float64)).to(dev)
        desc.reg_dev = rt.data_ptr()
        keep.append(rt)
    else:
        Rt = torch.from_numpy(np.ascontiguousarray(reg, dtype=np.complex128)).to(dev)
        desc.R_dev = Rt.data_ptr()
        keep.append(Rt)
    desc.lam = float(lam)
    L = nat.lib()
    ws = nat.workspace(L.fdl_solve_dense_workspace(desc), dev)
    nat.check(L.fdl_solve_dense(desc, ws.data_ptr(), ws.numel(), nat.stream_handle(dev)), "fdl_solve_dense")
    return x.cpu().numpy(), status.cpu().numpy()


def _reg_matrix(reg, n):
    """construct.py:112-120 (validation of the regulariser argument)."""
    reg = np.asarray(reg, dtype=np.float64) if np.isrealobj(reg) else np.asarray(reg)
    if reg.ndim == 1:
        if reg.shape != (n,):
            raise ValueError("diagonal regularizer length must equal layer count")
        return reg
    if reg.shape != (n, n):
        raise ValueError("regularizer must be an n-vector or n x n matrix")
    return reg


def solve_frequency(A, b, reg, lam: float, freq=None):
    """x = (A*A + lam reg)^-1 A*b for one frequency (construct.py:123-154), on the GPU.

    Same contract as the reference: the normal-equation residual is below
    1e-8 relative, a degenerate system with lam > 0 falls back to the
    minimum-norm stacked least squares, lam = 0 raises RankDeficiencyError
    when the system is singular or over-parameterised.
    """
    A = np.asarray(A, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    m, n = A.shape
    if lam < 0:
        raise ValueError("lam must be non-negative")
    if lam == 0 and n > m:
        raise RankDeficiencyError(f"{n} layers from {m} images is ill-posed without regularization")
    R = _reg_matrix(reg, n)
    vec = b.ndim == 1
    bb = b.reshape(m, -1)
    Rb = R[None] if R.ndim == 2 else R[None, :]
    x, status = solve_dense(A[None], bb[None], Rb, lam)
    tag = "" if freq is None else f" at frequency {freq}"
    if status[0] == 3:
        raise RankDeficiencyError(f"singular normal matrix{tag}")
    if status[0] == 1:
        raise nat.FdlNativeError(f"minimum-norm fallback failed{tag}")
    out = x[0]
    return out[:, 0] if vec else out


def default_lambda(b_norms_sq, m: int) -> float:
    """1e-4 * mean_q ||b_q||^2 / m (construct.py:214-216)."""
    return 1e-4 * float(np.mean(b_norms_sq)) / m


class ConstructStats:
    """What the last construct_fdl call on this thread did."""

    def __init__(self):
        self.path = 0              # K1 formulation: 1 symmetric-real, 2 real-A, 3 complex
        self.breakdown_bins = 0    # bins left unsolved
        self.fallback_bins = 0     # bins re-solved by the minimum-norm fallback
        self.audited_bins = 0      # bins the residual screen sent to the reference's exact test
        self.lam = None


import threading

_tls = threading.local()


def last_construct_stats() -> ConstructStats:
    st = getattr(_tls, "stats", None)
    if st is None:
        st = _tls.stats = ConstructStats()
    return st


def _require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1901_06919_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _views_device(images, device):
    """(m,H,W,C) float32 contiguous CUDA tensor."""
    import torch
    if _is_torch(images):
        t = images
    else:
        arr = np.ascontiguousarray(images, dtype=np.float32)
        t = torch.from_numpy(arr)
        if device.type == "cuda":
            t = t.pin_memory() if arr.nbytes >= (1 << 20) else t
    return t.to(device=device, dtype=torch.float32, non_blocking=True).contiguous()


def aperture_table_set(apertures):
    """Unique non-pinhole ApertureSpecs and per-view indices (-1 for pinholes)."""
    uniq, idx = [], []
    for ap in apertures:
        if ap is None or ap.is_pinhole:
            idx.append(-1)
            continue
        for i, u in enumerate(uniq):
            if u is ap:
                idx.append(i)
                break
        else:
            uniq.append(ap)
            idx.append(len(uniq) - 1)
    return uniq, np.asarray(idx, dtype=np.int32)


@nat.on_device(lambda spectra, *a, **k: spectra.device)
def solve_slab(spectra, m, n, C, Hp, Wp, rows, shifts_pu, shifts_pv, d, lam, eps, views=None,
               u=None, v=None, force_path=0, status=None, out=None, full_grid=False, count=True, lam_fn=None,
               lam_dev=None, chunk=None, chunk_sync=None, resolve_only=None, audit_only=None):
    """Run K1 on a slab of frequency rows; returns (layers (n,C,nrows,Whp) c64, n_breakdown, path).

    full_grid: spectra / out are full (.., Hp, Whp) buffers and only `rows` are
    solved, in place (plane_rows = Hp).  count=False skips the breakdown count
    (no host synchronisation; n_breakdown is returned as None and the caller
    inspects `status`).  lam_dev: a (1,) float64 CUDA tensor holding lambda
    (lambda_device): K1 reads it on the device, no host round trip; lam is
    then ignored.  lam_fn: lam is None and lam_fn() gives it (host).  chunk:
    the reference's solve chunk (fallback granularity, fallback_bins).
    audit_only: host array of slab bins -- skip K1 and run the reference's residual
    test on those (returns their verdicts in place of the breakdown count);
    resolve_only: host array of slab bins -- skip K1 and only re-solve those
    bins by the minimum-norm fallback (lam > 0), into `out`."""
    import torch
    device = spectra.device
    whp = Wp // 2 + 1
    nrows = len(rows)
    if chunk is None:
        chunk = SOLVE_CHUNK
    layers = out if out is not None else torch.empty((n, C, Hp if full_grid else nrows, whp),
                                                     dtype=torch.complex64, device=device)
    if status is None:
        status = torch.zeros((nrows, whp), dtype=torch.int8, device=device)
    rows_np = np.ascontiguousarray(rows, dtype=np.int32)
    d = np.ascontiguousarray(d, dtype=np.float64)
    keep = [rows_np, d]
    desc = nat.FdlSolveDesc()
    desc.m, desc.n, desc.C, desc.Hp, desc.Wp, desc.nrows = m, n, C, Hp, Wp, nrows
    desc.rows = nat.iptr(rows_np)
    if u is not None:
        u_ = np.ascontiguousarray(u, dtype=np.float64)
        v_ = np.ascontiguousarray(v, dtype=np.float64)
        keep += [u_, v_]
        desc.u, desc.v = nat.dptr(u_), nat.dptr(v_)
    else:
        pu_ = np.ascontiguousarray(shifts_pu, dtype=np.float64)
        pv_ = np.ascontiguousarray(shifts_pv, dtype=np.float64)
        keep += [pu_, pv_]
        desc.pu, desc.pv = nat.dptr(pu_), nat.dptr(pv_)
    desc.d = nat.dptr(d)
    if views is not None and not views.all_pinhole:
        uniq, idx = aperture_table_set(views.apertures)
        arr, keep_ap = nat.aperture_structs(uniq)
        s_ = np.ascontiguousarray(views.s, dtype=np.float64)
        sc_ = np.ascontiguousarray(views.aperture_scale, dtype=np.float64)
        keep += [idx, s_, sc_, arr, keep_ap]
        desc.view_aperture = nat.iptr(idx)
        desc.s, desc.scale = nat.dptr(s_), nat.dptr(sc_)
        desc.n_apertures = len(uniq)
        desc.apertures = arr
    desc.lam, desc.eps = (float(lam) if lam is not None else 0.0), float(eps)  # lam does not shape the plan
    desc.spectra_dev = spectra.data_ptr()
    desc.layers_dev = layers.data_ptr()
    desc.status_dev = status.data_ptr()
    desc.force_path = int(force_path)
    desc.plane_rows = Hp if full_grid else 0
    if lam_dev is not None:
        desc.lam_dev = lam_dev.data_ptr()
    L = nat.lib()
    path = L.fdl_solve_path(desc)
    if path < 0:
        nat.check(path, "fdl_solve_path")
    if resolve_only is not None:
        resolve_bins(desc, np.ascontiguousarray(resolve_only, dtype=np.int32), device)
        return layers, None, path
    if audit_only is not None:  # the residual test on FDL_BIN_SUSPECT bins -> their verdicts
        return layers, audit_bins(desc, np.ascontiguousarray(audit_only, dtype=np.int32), device), path
    ws_bytes = L.fdl_solve_bins_workspace(desc)
    if ws_bytes == 0:
        nat.check(L.fdl_solve_path(desc), "fdl_solve_bins_workspace")
    ws = nat.workspace(ws_bytes, device)
    nb = nat.ctypes.c_int32(0)
    if lam_fn is not None:
        lam = float(lam_fn())
        desc.lam = lam
    nat.check(L.fdl_solve_bins(desc, ws.data_ptr(), ws.numel(), nat.ctypes.byref(nb) if count else None,
                               nat.stream_handle(device)), "fdl_solve_bins")
    if not count:
        return layers, None, path
    n_bad = int(nb.value)
    if n_bad and lam_dev is not None:
        lam = float(lam_dev.item())
        desc.lam, desc.lam_dev = lam, None
    resolved = 0
    if n_bad:
        flags = status.cpu().numpy().reshape(-1)
        suspects = np.flatnonzero(flags == nat.FDL_BIN_SUSPECT)
        if suspects.size:
            # the reference's own residual test (construct.py:198-210) on the bins the screen
            # marked: accepted bins keep a normal-equation solve, failing bins are re-solved
            # by minimum-norm least squares one by one (lam = 0: they stay flagged and
            # construct_fdl raises RankDeficiencyError)
            verdicts = audit_bins(desc, suspects.astype(np.int32), device)
            last_construct_stats().audited_bins += int(suspects.size)
            resolved += int(np.count_nonzero(verdicts == 2))
            flags = status.cpu().numpy().reshape(-1)
        n_bad = int(np.count_nonzero(flags))
    if n_bad and lam > 0:
        bins = fallback_bins(flags, rows, whp, chunk, chunk_sync)
        resolve_bins(desc, bins, device)
        resolved += len(bins)
        n_bad = int(torch.count_nonzero(status).item())
    st = last_construct_stats()
    st.fallback_bins = resolved - n_bad
    return layers, n_bad, path


def fallback_bins(status_flat, rows, whp: int, chunk: int, chunk_sync=None):
    """Slab bins (row-major flat indices) the reference re-solves by minimum-norm
    least squares when K1 flagged `status_flat` != 0 (construct.py:196-210):
    np.linalg.solve raises for the WHOLE chunk of `chunk` consecutive bins
    (flat q = ky * Whp + kx, construct.py:277-284) that holds a singular normal
    matrix, and every bin of that chunk is re-solved.  chunk_sync (multi-GPU)
    merges the bad-chunk sets of all ranks, whose slabs may share a chunk."""
    rows = np.asarray(rows, dtype=np.int64)
    bad = np.flatnonzero(status_flat)
    gq = rows[bad // whp] * whp + bad % whp
    chunks = np.unique(gq // max(1, int(chunk)))
    if chunk_sync is not None:
        chunks = chunk_sync(chunks)
    allq = (rows[:, None] * whp + np.arange(whp)[None, :]).reshape(-1)
    return np.ascontiguousarray(np.flatnonzero(np.isin(allq // max(1, int(chunk)), chunks)), dtype=np.int32)


RESOLVE_BATCH = 4096  # bins per fdl_resolve_bins call (bounds the workspace: ~m n 16 B per bin)


def audit_bins(desc, bins, device):
    """The reference's per-bin acceptance test (construct.py:198-210) on the listed slab
    bins (fdl_audit_bins), in batches -> int8 verdicts: 0 normal equations accepted,
    2 minimum-norm fallback used, 1 fallback failed, 3 residual test failed at lam = 0."""
    L = nat.lib()
    out = np.zeros(len(bins), dtype=np.int8)
    for b0 in range(0, len(bins), RESOLVE_BATCH):
        part = np.ascontiguousarray(bins[b0:b0 + RESOLVE_BATCH], dtype=np.int32)
        verdict = np.zeros(len(part), dtype=np.int8)
        rws = nat.workspace(L.fdl_resolve_bins_workspace(desc, len(part)), device)
        nat.check(L.fdl_audit_bins(desc, nat.iptr(part), len(part), verdict.ctypes.data, rws.data_ptr(), rws.numel(),
                                   nat.stream_handle(device)), "fdl_audit_bins")
        out[b0:b0 + len(part)] = verdict
    return out


def resolve_bins(desc, bins, device):
    """The reference's minimum-norm fallback (construct.py:157-165) on the GPU for
    the listed slab bins, in batches."""
    L = nat.lib()
    for b0 in range(0, len(bins), RESOLVE_BATCH):
        part = np.ascontiguousarray(bins[b0:b0 + RESOLVE_BATCH], dtype=np.int32)
        rws = nat.workspace(L.fdl_resolve_bins_workspace(desc, len(part)), device)
        nat.check(L.fdl_resolve_bins(desc, nat.iptr(part), len(part), rws.data_ptr(), rws.numel(),
                                     nat.stream_handle(device)), "fdl_resolve_bins")


@nat.on_device(lambda views_dev, *a, **k: views_dev.device)
def views_to_spectra(views_dev, pad, srgb: bool = False):
    """K0 on a (m,H,W,C) float32 CUDA tensor -> (spectra (m,C,Hp,Whp) c64, per-view sum|b|^2 (m) f64).
    srgb: the views are sRGB-encoded and are decoded to linear light as K0 loads them."""
    import torch
    m, H, W, C = views_dev.shape
    Hp, Wp = H + 2 * pad, W + 2 * pad
    device = views_dev.device
    spectra = torch.empty((m, C, Hp, Wp // 2 + 1), dtype=torch.complex64, device=device)
    sumsq = torch.empty((m,), dtype=torch.float64, device=device)
    L = nat.lib()
    ws_bytes = L.fdl_views_to_spectra_workspace(m, H, W, C, pad)
    if ws_bytes == 0:
        raise nat.FdlNativeError("fdl_views_to_spectra_workspace: " + L.fdl_last_error().decode())
    ws = nat.workspace(ws_bytes, device)
    k0 = L.fdl_views_to_spectra_srgb if srgb else L.fdl_views_to_spectra
    nat.check(k0(views_dev.data_ptr(), m, H, W, C, pad, spectra.data_ptr(),
                 sumsq.data_ptr(), ws.data_ptr(), ws.numel(), nat.stream_handle(device)), "fdl_views_to_spectra")
    return spectra, sumsq


UPLOAD_CHUNK_BYTES = 24 << 20


@nat.on_device(lambda images, pad, device, *a, **k: device)
def views_to_spectra_host(images, pad, device, chunk_bytes: int = UPLOAD_CHUNK_BYTES, srgb: bool = False):
    """K0 on HOST views with the upload overlapped: view chunks go host->device
    on a side stream while K0 transforms the previous chunk on the current
    stream.  Pinned torch input is copied directly; anything else passes
    through a two-slot pinned staging ring.  K0 is batch-independent bit for
    bit (tests/test_gpu_sharded.py), so the result equals the one-shot call."""
    import torch
    quant = images if isinstance(images, QuantisedImages) else None
    if quant is not None:
        # 8- / 16-bit views cross PCIe quantised and are decoded on the device (fdl_dequantise_views)
        src = quant.torch_host()
    else:
        src = images if _is_torch(images) else torch.from_numpy(np.ascontiguousarray(images, dtype=np.float32))
        if src.dtype != torch.float32 or not src.is_contiguous():
            src = src.to(torch.float32).contiguous()
    m, H, W, C = src.shape
    Hp, Wp = H + 2 * pad, W + 2 * pad
    per = max(1, min(m, chunk_bytes // max(1, H * W * C * 4)))
    spectra = torch.empty((m, C, Hp, Wp // 2 + 1), dtype=torch.complex64, device=device)
    sumsq = torch.empty((m,), dtype=torch.float64, device=device)
    views_dev = torch.empty((m, H, W, C), dtype=torch.float32, device=device)
    L = nat.lib()
    ws_bytes = L.fdl_views_to_spectra_workspace(per, H, W, C, pad)
    if ws_bytes == 0:
        raise nat.FdlNativeError("fdl_views_to_spectra_workspace: " + L.fdl_last_error().decode())
    ws = nat.workspace(ws_bytes, device)
    compute = torch.cuda.current_stream(device)
    copy = nat.copy_stream(device)
    copy.wait_stream(compute)  # views_dev was allocated on the compute stream
    pinned = src.is_pinned()
    ring = [] if pinned else [torch.empty((per, H, W, C), dtype=src.dtype, pin_memory=True) for _ in range(2)]
    ring_ev = [None, None]
    # quantised input lands in its own device buffer and is decoded into views_dev on the compute stream
    land = torch.empty((m, H, W, C), dtype=src.dtype, device=device) if quant is not None else views_dev
    for i, j0 in enumerate(range(0, m, per)):
        j1 = min(m, j0 + per)
        with torch.cuda.stream(copy):
            if pinned:
                land[j0:j1].copy_(src[j0:j1], non_blocking=True)
            else:
                b = i % 2
                if ring_ev[b] is not None:
                    ring_ev[b].synchronize()  # the slot's previous H2D has drained
                ring[b][:j1 - j0].copy_(src[j0:j1])
                land[j0:j1].copy_(ring[b][:j1 - j0], non_blocking=True)
                ring_ev[b] = torch.cuda.Event()
                ring_ev[b].record(copy)
            ev = torch.cuda.Event()
            ev.record(copy)
        compute.wait_event(ev)
        if quant is not None:
            nat.check(L.fdl_dequantise_views(land[j0].data_ptr(), quant.bits, (j1 - j0) * H * W * C,
                                             views_dev[j0].data_ptr(), nat.stream_handle(device)),
                      "fdl_dequantise_views")
        k0 = L.fdl_views_to_spectra_srgb if srgb else L.fdl_views_to_spectra
        nat.check(k0(views_dev[j0].data_ptr(), j1 - j0, H, W, C, pad, spectra[j0].data_ptr(), sumsq[j0:].data_ptr(),
                     ws.data_ptr(), ws.numel(), nat.stream_handle(device)), "fdl_views_to_spectra")
    for e in ring_ev:
        if e is not None:
            e.synchronize()  # the staging ring may be reused by the caching host allocator
    return spectra, sumsq


@nat.on_device(lambda layers, *a, **k: layers.device)
def symmetrize(layers, Hp, Wp, rows=None, mirror=None):
    n, C, nrows, _ = layers.shape
    L = nat.lib()
    r = np.ascontiguousarray(rows, dtype=np.int32) if rows is not None else None
    mi = np.ascontiguousarray(mirror, dtype=np.int32) if mirror is not None else None
    nat.check(L.fdl_symmetrize(layers.data_ptr(), n, C, Hp, Wp, nrows, nat.iptr(r), nat.iptr(mi),
                               nat.stream_handle(layers.device)), "fdl_symmetrize")


def resolve_shifts(views: ViewSet, shifts: ShiftParams):
    """Validation of construct.py:234-248; returns (pu, pv, d)."""
    pu, pv = shifts.expand()
    m = views.num_views
    if pu.shape[0] != m:
        raise ValueError(f"shift parameters describe {pu.shape[0]} views, got {m}")
    if shifts.d is None:
        raise ValueError("relaxed shift parameters need layer disparities attached")
    d = np.asarray(shifts.d, dtype=np.float64)
    return pu, pv, d


def default_pad_margin(pu, pv) -> int:
    """ceil(max |P|) (construct.py:250-252)."""
    if pu.size == 0:
        return 0
    return int(math.ceil(max(np.max(np.abs(pu)), np.max(np.abs(pv)))))


def lambda_device(view_sumsq_dev, Q: int, m: int):
    """default_lambda on the device (fdl_default_lambda): a (1,) float64 CUDA
    tensor, bit-identical to lambda_from_sumsq of the same sums."""
    import torch
    lam = torch.empty((1,), dtype=torch.float64, device=view_sumsq_dev.device)
    nat.check(nat.lib().fdl_default_lambda(view_sumsq_dev.data_ptr(), m, int(Q), lam.data_ptr(),
                                           nat.stream_handle(view_sumsq_dev.device)), "fdl_default_lambda")
    return lam


def lambda_from_sumsq(view_sumsq, Q: int, m: int) -> float:
    """default_lambda from per-view partial sums, summed on the host in view order."""
    tot = 0.0
    for s in np.asarray(view_sumsq, dtype=np.float64):
        tot += float(s)
    return 1e-4 * (tot / Q) / m


@nat.on_device(lambda views, shifts, *a, device=None, **k: device)
def construct_fdl(views: ViewSet, shifts: ShiftParams, lam: float | None = None, eps: float = DEFAULT_EPS,
                  pad_margin: int | None = None, chunk: int = SOLVE_CHUNK, *, device=None,
                  force_path: int = 0, eager_host: bool | None = None, decode_srgb: bool = False) -> FdlModel:
    """Build the disparity-layer model by per-frequency solves (construct.py:219-308).

    Same arguments, defaults and exceptions as the reference.  Every bin is
    solved independently in one launch; `chunk` only sets the reference's
    fallback granularity (a singular bin sends its whole chunk of `chunk`
    bins to the minimum-norm solve, construct.py:196-210).  `device` picks the CUDA device (default:
    current); `force_path` pins the K1 formulation (testing).  `eager_host`
    (default: when the views came from host memory) reads the layers back to
    pinned host memory slab by slab while later slabs solve; the model's
    `.layers` / `layers_host()` then need no further transfer.  `decode_srgb`
    (gamma-encoded views only) builds the model in linear light, decoding
    every value as K0 loads it: the reference's load_lightfield(...,
    to_linear=True) + construct_fdl (io.py:147-149) without a decoded copy.
    """
    if decode_srgb and views.color_space != GAMMA:
        raise ValueError("decode_srgb needs gamma-encoded (sRGB) views")
    torch = _require_cuda()
    last_construct_stats().fallback_bins = 0
    last_construct_stats().audited_bins = 0
    pu, pv, d = resolve_shifts(views, shifts)
    m = views.num_views
    n = pu.shape[1]
    if lam == 0 and n > m:
        raise RankDeficiencyError(f"{n} layers from {m} images is ill-posed without regularization")
    if pad_margin is None:
        pad_margin = default_pad_margin(pu, pv)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    H, W, C = views.height, views.width, views.channels
    Hp, Wp = H + 2 * pad_margin, W + 2 * pad_margin
    grid = FrequencyGrid(width=Wp, height=Hp)
    if _is_torch(views.images) and views.images.is_cuda:
        spectra, sumsq = views_to_spectra(_views_device(views.images, dev), pad_margin, srgb=decode_srgb)
    else:
        spectra, sumsq = views_to_spectra_host(views.images, pad_margin, dev, srgb=decode_srgb)
    if eager_host is None:
        eager_host = not (_is_torch(views.images) and views.images.is_cuda)
    pipelined = eager_host and Hp >= 4 * PIPELINE_SLABS
    if lam is not None and lam < 0:
        raise ValueError("lam must be non-negative")
    # the default lambda stays on the device (no host round trip between K0 and K1)
    lam_dev = lambda_device(sumsq, grid.num_entries, m) if lam is None else None
    u = views_u = None
    if shifts.is_factored:
        u, views_u = shifts.u, shifts.v
    host = None
    if pipelined:
        layers, host, path = _solve_pipelined(spectra, m, n, C, Hp, Wp, pu, pv, d, lam, eps, views, u, views_u,
                                              force_path, lam_dev)
        n_bad = 0
        if host is None:  # some bin broke down: the plain path below re-solves with the fallback
            layers = None
    if host is None:
        layers, n_bad, path = solve_slab(spectra, m, n, C, Hp, Wp, np.arange(Hp), pu, pv, d, lam, eps,
                                         views=views, u=u, v=views_u, force_path=force_path, lam_dev=lam_dev,
                                         chunk=chunk)
    if lam is None:
        lam = float(lam_dev.item())
    st = last_construct_stats()
    st.path, st.breakdown_bins, st.lam = path, n_bad, float(lam)
    if n_bad:
        if lam == 0:
            raise RankDeficiencyError("singular normal matrix at some frequency")
        raise nat.FdlNativeError(f"{n_bad} bins could not be solved (minimum-norm fallback failed)")
    if host is None:
        symmetrize(layers, Hp, Wp)
    model = FdlModel(disparities=d, layers=layers, grid=grid, width=W, height=H, pad_margin=pad_margin,
                     color_space=LINEAR if decode_srgb else views.color_space, calibration=shifts,
                     lambda_used=float(lam))
    if host is not None:
        model._host_async = host
    return model


PIPELINE_SLABS = 4  # conjugate-row slabs of the overlapped read-back


def _row_runs(rows):
    """Maximal runs [a, b) of consecutive values of a sorted row list."""
    runs, a = [], int(rows[0])
    for x, y in zip(rows[:-1], rows[1:]):
        if int(y) != int(x) + 1:
            runs.append((a, int(x) + 1))
            a = int(y)
    runs.append((a, int(rows[-1]) + 1))
    return runs


@nat.on_device(lambda spectra, *a, **k: spectra.device)
def _solve_pipelined(spectra, m, n, C, Hp, Wp, pu, pv, d, lam, eps, views, u, v, force_path, lam_dev=None):
    """K1 + K2 in PIPELINE_SLABS slabs of conjugate row pairs, each slab's
    finished rows copied to pinned host memory on a side stream while the next
    slab solves (the reference returns host layers, construct.py:300-308).
    Returns (device layers, (host tensor, event), path), or (layers, None, path)
    when a bin broke down (the caller re-solves with the fallback)."""
    import torch
    from .dist import slab_rows
    device = spectra.device
    whp = Wp // 2 + 1
    layers = torch.empty((n, C, Hp, whp), dtype=torch.complex64, device=device)
    host = torch.empty((n, C, Hp, whp), dtype=torch.complex64, pin_memory=True)
    compute = torch.cuda.current_stream(device)
    copy = nat.copy_stream(device)
    L = nat.lib()
    statuses, path = [], 0
    for s_ in range(PIPELINE_SLABS):
        rows, _ = slab_rows(Hp, PIPELINE_SLABS, s_)
        if len(rows) == 0:
            continue
        status = torch.zeros((len(rows), whp), dtype=torch.int8, device=device)
        statuses.append(status)
        _, _, path = solve_slab(spectra, m, n, C, Hp, Wp, rows, pu, pv, d, lam, eps, views=views, u=u, v=v,
                                force_path=force_path, status=status, out=layers, full_grid=True, count=False,
                                lam_dev=lam_dev)
        r32 = np.ascontiguousarray(rows, dtype=np.int32)
        nat.check(L.fdl_symmetrize_rows(layers.data_ptr(), n, C, Hp, Wp, len(r32), nat.iptr(r32),
                                        nat.stream_handle(device)), "fdl_symmetrize_rows")
        ev = torch.cuda.Event()
        ev.record(compute)
        copy.wait_event(ev)
        for a, b in _row_runs(r32):
            nat.check(L.fdl_rows_to_host(layers.data_ptr(), host.data_ptr(), n * C, Hp, whp, a, b,
                                         nat.ctypes.c_void_p(copy.cuda_stream)), "fdl_rows_to_host")
    done = torch.cuda.Event()
    done.record(copy)
    layers.record_stream(copy)
    if any(int(torch.count_nonzero(st_).item()) for st_ in statuses):
        done.synchronize()
        return layers, None, path
    return layers, (host, done), path

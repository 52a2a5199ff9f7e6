"""Rendering from a disparity-layer model on the B200 (reference: fdl/render.py).

`render(model, req)` keeps the reference signature, validation, side effects
(`last_render_stats()`, `ApertureSpec.oob_count`) and output (float64 numpy,
(H, W) or (H, W, C)).  The work is two native stages:

  K3 fdl_render_spectra     per-bin weighted layer sum          (render.py:190-207, lfmodel.py:101-122)
  K4 fdl_spectra_to_images  cuFFT C2R + crop + optional sRGB    (spectra.py:202-208, render.py:210-225)

`render_many(model, reqs)` is the batched form (one K3 launch per batch of
views, one K4 per batch) that the benchmarks and `render_views_with_shifts`
use; `render` is its V = 1 case.  Statistics are kept per thread, so the
concurrent HTTP callers of the reference's serve.py:115-143 do not race on a
shared global (the reference's `_LAST_STATS` is module-global, render.py:183).
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .lfmodel import LINEAR, ApertureSpec, FdlModel

__all__ = [
    "RenderRequest",
    "RenderStats",
    "aperture_spectrum",
    "render",
    "render_many",
    "render_views_with_shifts",
    "srgb_encode",
    "srgb_decode",
    "last_render_stats",
]

DEFAULT_PAD_FACTOR = 4     # render.py:34
DEFAULT_RESOLUTION = 64    # render.py:35
_SUPERSAMPLE = 4           # render.py:36


def srgb_decode(x):
    """sRGB -> linear light (render.py:39-42)."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x <= 0.04045, x / 12.92, ((np.clip(x, 0.04045, None) + 0.055) / 1.055) ** 2.4)


def srgb_encode(x):
    """Linear light -> sRGB, negatives clamp to 0 (render.py:45-48)."""
    x = np.clip(np.asarray(x, dtype=np.float64), 0.0, None)
    return np.where(x <= 0.0031308, x * 12.92, 1.055 * np.clip(x, 0.0031308, None) ** (1 / 2.4) - 0.055)


def _coverage(shape: str, resolution: int, **params):
    """(coverage raster, physical extent) of an aperture shape (render.py:51-90)."""
    fine = resolution * _SUPERSAMPLE
    if shape == "square":
        side = float(params["side"])
        if side <= 0:
            raise ValueError("square aperture needs a positive side")
        return np.ones((resolution, resolution)), side
    if shape == "disk":
        diameter = float(params["diameter"])
        if diameter <= 0:
            raise ValueError("disk aperture needs a positive diameter")
        ctr = np.arange(fine) + 0.5 - fine / 2
        inside = (ctr[None, :] ** 2 + ctr[:, None] ** 2) <= (fine / 2) ** 2
        return inside.reshape(resolution, _SUPERSAMPLE, resolution, _SUPERSAMPLE).mean(axis=(1, 3)), diameter
    if shape == "polygon":
        verts = np.asarray(params["vertices"], dtype=np.float64)
        if verts.ndim != 2 or verts.shape[0] < 3 or verts.shape[1] != 2:
            raise ValueError("polygon aperture needs at least 3 (x, y) vertices")
        from PIL import Image, ImageDraw
        extent = 2.0 * float(np.max(np.abs(verts)))
        if extent <= 0:
            raise ValueError("invalid aperture: zero area")
        canvas = Image.new("L", (fine, fine), 0)
        xs = (verts[:, 0] / extent + 0.5) * fine - 0.5
        ys = (verts[:, 1] / extent + 0.5) * fine - 0.5
        ImageDraw.Draw(canvas).polygon(list(zip(xs.tolist(), ys.tolist())), fill=255)
        cov = np.asarray(canvas, dtype=np.float64) / 255.0
        return cov.reshape(resolution, _SUPERSAMPLE, resolution, _SUPERSAMPLE).mean(axis=(1, 3)), extent
    if shape == "raster":
        img = np.asarray(params["image"], dtype=np.float64)
        if img.ndim != 2 or img.size == 0:
            raise ValueError("raster aperture needs a 2D image")
        return img, float(params["extent"])
    raise ValueError(f"unknown aperture shape {shape!r}")


def aperture_spectrum(shape: str, pad_factor: int = DEFAULT_PAD_FACTOR,
                      resolution: int = DEFAULT_RESOLUTION, **params) -> ApertureSpec:
    """Sampled, area-normalised aperture spectrum (render.py:93-132).

    Built once per aperture on the host (a 256x256 table by default) and
    uploaded to the device by the kernels that use it; not a hot-path op.
    """
    if pad_factor < 1:
        raise ValueError("pad_factor must be >= 1")
    if shape == "pinhole":
        return ApertureSpec(shape="pinhole", pad_factor=pad_factor)
    raster, extent = _coverage(shape, resolution, **params)
    area = raster.sum()
    if area <= 0:
        raise ValueError("invalid aperture: zero area")
    nr, nc = raster.shape
    if extent <= 0:
        raise ValueError("aperture extent must be positive")
    du = extent / max(nr, nc)
    big = np.zeros((nr * pad_factor, nc * pad_factor))
    big[:nr, :nc] = raster
    spec = np.fft.fft2(big)
    # centre the pixel grid on the physical origin
    spec *= (np.exp(2j * np.pi * np.fft.fftfreq(nr * pad_factor) * ((nr - 1) / 2))[:, None]
             * np.exp(2j * np.pi * np.fft.fftfreq(nc * pad_factor) * ((nc - 1) / 2))[None, :])
    table = np.fft.fftshift(spec) / area
    xi_x = np.fft.fftshift(np.fft.fftfreq(nc * pad_factor, d=du))
    xi_y = np.fft.fftshift(np.fft.fftfreq(nr * pad_factor, d=du))
    if np.max(np.abs(table.imag)) < 1e-12 * np.max(np.abs(table.real)):
        table = np.ascontiguousarray(table.real)
    label = {"square": f"square({params.get('side')})", "disk": f"disk({params.get('diameter')})",
             "polygon": "polygon", "raster": "raster"}[shape]
    return ApertureSpec(shape=label, pad_factor=pad_factor, table=table, xi_x=xi_x, xi_y=xi_y)


@dataclass
class RenderRequest:
    """Viewpoint (u, v), refocus s, aperture scale f >= 0 (render.py:135-160)."""

    u: float = 0.0
    v: float = 0.0
    s: float = 0.0
    f: float = 0.0
    aperture: ApertureSpec | None = None
    gamma_mode: str = "as-stored"
    crop: bool = True

    def __post_init__(self):
        if not np.isfinite(self.u) or not np.isfinite(self.v):
            raise ValueError("u and v must be finite")
        if not np.isfinite(self.s):
            raise ValueError("s must be finite")
        if not (np.isfinite(self.f) and self.f >= 0):
            raise ValueError("f must be >= 0")
        if self.gamma_mode not in ("as-stored", "linear-process"):
            raise ValueError(f"unknown gamma_mode {self.gamma_mode!r}")


@dataclass
class RenderStats:
    """Operation count of the last render on this thread (render.py:163-187)."""

    layer_ops: int = 0
    num_layers: int = 0
    grid_bins: int = 0
    seconds: float = 0.0
    aperture_pass: bool = False
    oob_lookups: int = 0

    def reset(self):
        self.layer_ops = 0
        self.num_layers = 0
        self.grid_bins = 0
        self.seconds = 0.0
        self.aperture_pass = False
        self.oob_lookups = 0


_tls = threading.local()


def last_render_stats() -> RenderStats:
    st = getattr(_tls, "stats", None)
    if st is None:
        st = _tls.stats = RenderStats()
    return st


def _uses_aperture(req: RenderRequest) -> bool:
    # render.py:240: the aperture pass runs iff f > 0 and the aperture is not a pinhole
    return req.f > 0 and req.aperture is not None and not req.aperture.is_pinhole


@nat.on_device(lambda layers_dev, *a, **k: layers_dev.device)
def render_spectra_batch(layers_dev, d, Hp, Wp, pu, pv, t=None, view_ap=None, apertures=(), oob=None,
                         start_event=None):
    """K3 over V views -> (V, C, Hp, Whp) complex64 CUDA tensor."""
    import torch
    n, C = layers_dev.shape[0], layers_dev.shape[1]
    V = pu.shape[0]
    out = torch.empty((V, C, Hp, Wp // 2 + 1), dtype=torch.complex64, device=layers_dev.device)
    d = np.ascontiguousarray(d, dtype=np.float64)
    pu = np.ascontiguousarray(pu, dtype=np.float64)
    pv = np.ascontiguousarray(pv, dtype=np.float64)
    keep = [d, pu, pv]
    desc = nat.FdlRenderDesc()
    desc.n, desc.C, desc.Hp, desc.Wp, desc.V = n, C, Hp, Wp, V
    desc.d, desc.pu, desc.pv = nat.dptr(d), nat.dptr(pu), nat.dptr(pv)
    if view_ap is not None and len(apertures):
        t = np.ascontiguousarray(t, dtype=np.float64)
        va = np.ascontiguousarray(view_ap, dtype=np.int32)
        arr, keep_ap = nat.aperture_structs(list(apertures))
        keep += [t, va, arr, keep_ap]
        desc.t = nat.dptr(t)
        desc.view_aperture = nat.iptr(va)
        desc.n_apertures = len(apertures)
        desc.apertures = arr
    desc.layers_dev = layers_dev.data_ptr()
    desc.out_dev = out.data_ptr()
    desc.oob_dev = oob.data_ptr() if oob is not None else None
    L = nat.lib()
    # O(1) bound (fdl_render_spectra plans the batch once; the exact
    # fdl_render_workspace would scan it a second time on the host)
    entries = sum(int(np.asarray(a.table).shape[0]) * int(np.asarray(a.table).shape[1]) for a in apertures)
    ws_bytes = L.fdl_render_workspace_bound(n, C, Hp, Wp, V, len(apertures), entries)
    if ws_bytes == 0:
        raise nat.FdlNativeError("fdl_render_workspace_bound: invalid render shape")
    ws = nat.workspace(ws_bytes, layers_dev.device)
    if start_event is not None:  # stage timing: device work only, after the Python-side preparation
        start_event.record()
    nat.check(L.fdl_render_spectra(desc, ws.data_ptr(), ws.numel(), nat.stream_handle(layers_dev.device)),
              "fdl_render_spectra")
    return out


@nat.on_device(lambda spec, *a, **k: spec.device)
def spectra_to_images(spec, Hp, Wp, pad, Ho, Wo, srgb=False):
    """K4: (V, C, Hp, Whp) complex64 (destroyed) -> (V, Ho, Wo, C) float32 CUDA tensor."""
    import torch
    V, C = spec.shape[0], spec.shape[1]
    img = torch.empty((V, Ho, Wo, C), dtype=torch.float32, device=spec.device)
    L = nat.lib()
    ws_bytes = L.fdl_spectra_to_images_workspace(V, C, Hp, Wp)
    if ws_bytes == 0:
        raise nat.FdlNativeError("fdl_spectra_to_images_workspace: " + L.fdl_last_error().decode())
    ws = nat.workspace(ws_bytes, spec.device)
    nat.check(L.fdl_spectra_to_images(spec.data_ptr(), V, C, Hp, Wp, pad, Ho, Wo, int(bool(srgb)),
                                      img.data_ptr(), ws.data_ptr(), ws.numel(),
                                      nat.stream_handle(spec.device)), "fdl_spectra_to_images")
    return img


def _check_gamma(model: FdlModel, req: RenderRequest):
    if req.gamma_mode == "linear-process" and model.color_space != LINEAR:
        raise ValueError("linear-process rendering needs a model built in linear light "
                         f"(model stores {model.color_space!r} data)")


@nat.on_device(lambda model, *a, **k: model.device)
def render_many_device(model: FdlModel, reqs, batch: int = 64, timing=None, on_batch=None):
    """Render requests to a (V, H, W, C) float32 CUDA tensor (cropped per req.crop,
    which must agree across the batch) plus per-view OOB counts.  Device-resident
    form of `render_many`; no host round trip besides the OOB counts."""
    import torch
    reqs = list(reqs)
    for r in reqs:
        _check_gamma(model, r)
    if not reqs:
        raise ValueError("no render requests")
    crop = reqs[0].crop
    if any(r.crop != crop for r in reqs):
        raise ValueError("render_many needs one crop mode per batch")
    srgb = [r.gamma_mode == "linear-process" for r in reqs]
    layers = model.layers_device()
    d = model.disparities
    Hp, Wp = model.grid.height, model.grid.width
    pad = model.pad_margin if crop else 0
    Ho = model.height if (crop and model.pad_margin) else Hp
    Wo = model.width if (crop and model.pad_margin) else Wp
    n, C = layers.shape[0], layers.shape[1]
    out = torch.empty((len(reqs), Ho, Wo, C), dtype=torch.float32, device=layers.device)
    oob = torch.zeros((len(reqs),), dtype=torch.int64, device=layers.device)
    for idx in _kernel_groups(reqs, batch):
        chunk = [reqs[i] for i in idx]
        V = len(chunk)
        contiguous = idx[-1] - idx[0] == V - 1
        u = np.array([r.u for r in chunk], dtype=np.float64)
        v = np.array([r.v for r in chunk], dtype=np.float64)
        pu = u[:, None] * d[None, :]
        pv = v[:, None] * d[None, :]
        aps, view_ap = [], np.full(V, -1, dtype=np.int32)
        t = np.zeros((V, n))
        for i, r in enumerate(chunk):
            if _uses_aperture(r):
                for a, ap in enumerate(aps):
                    if ap is r.aperture:
                        view_ap[i] = a
                        break
                else:
                    aps.append(r.aperture)
                    view_ap[i] = len(aps) - 1
                t[i] = r.f * (r.s - d)
        evs = None
        if timing is not None:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        c_oob = oob[idx[0]:idx[0] + V] if contiguous else torch.zeros((V,), dtype=torch.int64, device=layers.device)
        spec = render_spectra_batch(layers, d, Hp, Wp, pu, pv, t=t,
                                    view_ap=view_ap if aps else None, apertures=aps, oob=c_oob,
                                    start_event=evs[0] if evs else None)
        if evs is not None:
            evs[1].record()
        flags = [srgb[i] for i in idx]
        if all(flags) or not any(flags):
            imgs = spectra_to_images(spec, Hp, Wp, pad, Ho, Wo, srgb=flags[0])
        else:
            imgs = torch.cat([spectra_to_images(spec[i:i + 1].contiguous(), Hp, Wp, pad, Ho, Wo, srgb=flags[i])
                              for i in range(V)])
        if evs is not None:
            evs[2].record()
            timing.append(evs)
        if contiguous:
            out[idx[0]:idx[0] + V] = imgs
            if on_batch is not None:
                on_batch(idx[0], V, out[idx[0]:idx[0] + V])
        else:
            it = torch.as_tensor(idx, device=layers.device)
            out.index_copy_(0, it, imgs)
            oob.index_copy_(0, it, c_oob)
            if on_batch is not None:
                for i in idx:
                    on_batch(i, 1, out[i:i + 1])
    return out, oob


def _kernel_groups(reqs, batch):
    """Request indices in K3 launches of <= `batch` views.  Views are grouped by
    the render tile they need (pinhole / real aperture table / complex table),
    so a view's image never depends on which other views share its launch
    (render_many(...)[i] == render(reqs[i]) bit for bit)."""
    def kind(r):
        if not _uses_aperture(r):
            return 0
        return 2 if np.iscomplexobj(r.aperture.table) else 1
    kinds = [kind(r) for r in reqs]
    if len(set(kinds)) == 1:
        return [list(range(b0, min(b0 + batch, len(reqs)))) for b0 in range(0, len(reqs), batch)]
    groups = []
    for k in sorted(set(kinds)):
        members = [i for i, kk in enumerate(kinds) if kk == k]
        groups += [members[b0:b0 + batch] for b0 in range(0, len(members), batch)]
    return groups


def _to_numpy_images(imgs, dtype=np.float64):
    """CUDA (V,H,W,C) float32 -> numpy (V,H,W[,C]) of `dtype`: cast on the device,
    one D2H copy into pinned memory (torch's caching host allocator), no host
    conversion pass."""
    import torch
    tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
    dev = imgs.to(tdt)
    host = torch.empty(dev.shape, dtype=tdt, pin_memory=True)
    host.copy_(dev, non_blocking=True)
    torch.cuda.current_stream(imgs.device).synchronize()
    arr = host.numpy()
    if arr.shape[-1] == 1:
        arr = arr[..., 0]
    return arr


def render_many(model: FdlModel, reqs, batch: int = 64, dtype=np.float64) -> list[np.ndarray]:
    """Batched `render`: one image per request (float64 like the reference, or
    float32 with dtype=np.float32); stats describe the last request."""
    t0 = time.perf_counter()
    reqs = list(reqs)
    import torch
    tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
    host_t, copy = None, None

    def drain(b0, V, dev_imgs):
        # cast this batch on the compute stream, read it back on the copy
        # stream while the next batch renders
        nonlocal host_t, copy
        if host_t is None:
            host_t = torch.empty((len(reqs),) + tuple(dev_imgs.shape[1:]), dtype=tdt, pin_memory=True)
            copy = nat.copy_stream(dev_imgs.device)
        cast = dev_imgs.to(tdt)
        ev = torch.cuda.Event()
        ev.record()
        copy.wait_event(ev)
        with torch.cuda.stream(copy):
            host_t[b0:b0 + V].copy_(cast, non_blocking=True)
        cast.record_stream(copy)

    _, oob = render_many_device(model, reqs, batch, on_batch=drain)
    copy.synchronize()
    host = host_t.numpy()
    if host.shape[-1] == 1:
        host = host[..., 0]
    oob_h = oob.cpu().numpy()
    for r, cnt in zip(reqs, oob_h):
        if _uses_aperture(r):
            r.aperture.add_oob(int(cnt))
    st = last_render_stats()
    st.reset()
    last = reqs[-1]
    q = model.grid.num_entries
    st.num_layers = model.num_layers
    st.grid_bins = q
    st.aperture_pass = _uses_aperture(last)
    st.layer_ops = model.num_layers * q * (3 if st.aperture_pass else 2)
    st.oob_lookups = int(oob_h[-1]) if st.aperture_pass else 0
    st.seconds = time.perf_counter() - t0
    return list(host)


def render(model: FdlModel, req: RenderRequest) -> np.ndarray:
    """Render one view (render.py:228-248): (H, W) or (H, W, C) float64."""
    return render_many(model, [req])[0]


def render_views_with_shifts(model: FdlModel, shifts) -> np.ndarray:
    """Pinhole views with explicit per-(view, layer) shifts (render.py:251-263): (m, H, W[, C])."""
    return _to_numpy_images(render_shifts_device(model, shifts))


@nat.on_device(lambda model, *a, **k: model.device)
def render_shifts_device(model: FdlModel, shifts):
    """`render_views_with_shifts` without the read-back: (m, H, W, C) float32 CUDA tensor."""
    pu, pv = shifts.expand()
    layers = model.layers_device()
    Hp, Wp = model.grid.height, model.grid.width
    pad = model.pad_margin
    Ho = model.height if pad else Hp
    Wo = model.width if pad else Wp
    spec = render_spectra_batch(layers, model.disparities, Hp, Wp, np.asarray(pu), np.asarray(pv))
    return spectra_to_images(spec, Hp, Wp, pad, Ho, Wo)

"""Seeded synthetic light fields for the five BASELINE.json configs (harness, not product).

SURVEY.md §8(d) fixes the generator; the reference's own generator
(`fdl/lfmodel.py:321-407`, `synthesize_lightfield`) cannot make occluded
scenes (its masks must partition the image, `lfmodel.py:333-341`), so the
harness writes its own:

* texture  : N(0,1) white noise -> Gaussian low-pass (transfer
             exp(-2 pi^2 sigma^2 |w|^2)) -> min-max normalised to [0,1]
             (per plane, per channel);
* mask     : Bernoulli(1/2) field, low-passed with sigma_m = 4 px, thresholded
             at its 70th percentile (30 % coverage); the farthest plane
             (smallest d) is a full-coverage background;
* composite: back-to-front in ascending d;
* shift    : plane content displaced by (-u d, -v d) px (the reference
             convention, `lfmodel.py:3-5`), a circular Fourier shift with the
             symmetric cosine value on even-size Nyquist lines
             (`spectra.py:211-221`), applied to texture and mask; the shifted
             mask is clipped to [0,1];
* noise    : N(0, sigma_n^2), views stored as float32, not clipped;
* order    : row-major, v outer and u inner (`tests/conftest.py:29-31`).

Everything runs in torch float64 on any device, so the same code makes the
small CPU test cases and the full-size B200 bench inputs.  All random draws
come from one `torch.Generator` seeded with the config number (C1..C5 ->
seeds 1..5); CPU and CUDA generators give different (equally valid) draws.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

__all__ = [
    "grid_coords",
    "LightFieldCase",
    "make_case",
    "CONFIG_NAMES",
    "random_fdl_layers",
    "render_requests_c5",
]

CONFIG_NAMES = ("c1", "c2", "c2b", "c3", "c4", "c5")


def grid_coords(side: int, spacing: float = 1.0, offset: float = 0.0) -> np.ndarray:
    """(side*side, 2) angular positions, v outer and u inner."""
    g = (np.arange(side) - (side - 1) / 2) * spacing + offset
    return np.array([(u, v) for v in g for u in g], dtype=np.float64)


def _freqs(h: int, w: int, device):
    fy = torch.fft.fftfreq(h, dtype=torch.float64, device=device)
    fx = torch.fft.rfftfreq(w, dtype=torch.float64, device=device)
    return fy, fx


def _lowpass(field_: torch.Tensor, sigma: float) -> torch.Tensor:
    h, w = field_.shape[-2:]
    fy, fx = _freqs(h, w, field_.device)
    tf = torch.exp(-2.0 * math.pi**2 * sigma**2 * (fy[:, None] ** 2 + fx[None, :] ** 2))
    return torch.fft.irfft2(torch.fft.rfft2(field_) * tf, s=(h, w))


def _minmax(x: torch.Tensor) -> torch.Tensor:
    flat = x.reshape(x.shape[0], -1) if x.dim() > 2 else x.reshape(1, -1)
    lo = flat.min(dim=1).values
    hi = flat.max(dim=1).values
    shape = (-1,) + (1,) * (x.dim() - 1) if x.dim() > 2 else ()
    return (x - lo.reshape(shape)) / (hi - lo).reshape(shape)


def _shift_phase(h: int, w: int, dx: torch.Tensor, dy: torch.Tensor, device) -> torch.Tensor:
    """(V, h, w//2+1) phase moving content by (+dx, +dy) px; cosine on Nyquist lines."""
    fy, fx = _freqs(h, w, device)
    ph_x = torch.exp(-2j * math.pi * fx[None, :] * dx[:, None])
    ph_y = torch.exp(-2j * math.pi * fy[None, :] * dy[:, None])
    if w % 2 == 0:
        ph_x[:, w // 2] = torch.cos(math.pi * dx).to(ph_x.dtype)
    if h % 2 == 0:
        ph_y[:, h // 2] = torch.cos(math.pi * dy).to(ph_y.dtype)
    return ph_y[:, :, None] * ph_x[:, None, :]


@dataclass
class LightFieldCase:
    """One synthetic input set plus everything needed to build and render it."""

    name: str
    views: torch.Tensor                 # (m, H, W, C) float32
    u: np.ndarray
    v: np.ndarray
    d: np.ndarray                       # layer disparities (strictly increasing)
    s: np.ndarray | None = None          # focal-stack refocus parameters
    aperture: dict | None = None         # {"shape": "disk", "diameter": ...} for every view
    render_coords: np.ndarray | None = None
    meta: dict = field(default_factory=dict)


def _planes(gen, n_planes, c, h, w, sigma, device):
    tex = torch.randn((n_planes, c, h, w), generator=gen, dtype=torch.float64, device=device)
    tex = _lowpass(tex, sigma)
    tex = _minmax(tex.reshape(n_planes * c, h, w)).reshape(n_planes, c, h, w)
    bern = (torch.rand((n_planes, h, w), generator=gen, dtype=torch.float64, device=device) < 0.5)
    blob = _lowpass(bern.to(torch.float64), 4.0)
    masks = torch.empty_like(blob)
    for p in range(n_planes):
        flat = blob[p].reshape(-1)
        k = int(math.ceil(0.7 * flat.numel()))
        thr = torch.kthvalue(flat.cpu(), k).values.to(device)
        masks[p] = (blob[p] > thr).to(torch.float64)
    masks[0] = 1.0  # farthest plane = full-coverage background
    return tex, masks


def _composite(tex, masks, plane_d, coords, chunk=16):
    """(m, C, H, W) float64 views of back-to-front composited shifted planes."""
    n_planes, c, h, w = tex.shape
    device = tex.device
    order = np.argsort(plane_d, kind="stable")
    tex_f = torch.fft.rfft2(tex)
    mask_f = torch.fft.rfft2(masks)
    cu = torch.as_tensor(coords[:, 0], dtype=torch.float64, device=device)
    cv = torch.as_tensor(coords[:, 1], dtype=torch.float64, device=device)
    out = torch.empty((len(coords), c, h, w), dtype=torch.float64, device=device)
    for j0 in range(0, len(coords), chunk):
        j1 = min(j0 + chunk, len(coords))
        acc = torch.zeros((j1 - j0, c, h, w), dtype=torch.float64, device=device)
        for p in order:
            dp = float(plane_d[p])
            ph = _shift_phase(h, w, -cu[j0:j1] * dp, -cv[j0:j1] * dp, device)
            t = torch.fft.irfft2(tex_f[p][None] * ph[:, None], s=(h, w))
            msk = torch.fft.irfft2(mask_f[p][None] * ph, s=(h, w)).clamp_(0.0, 1.0)[:, None]
            acc = t * msk + acc * (1.0 - msk)
        out[j0:j1] = acc
    return out


def _finish(views64, gen, noise):
    noise_t = torch.randn(views64.shape, generator=gen, dtype=torch.float64, device=views64.device)
    return (views64 + noise * noise_t).permute(0, 2, 3, 1).contiguous().to(torch.float32)


def make_case(name: str, size: int | tuple[int, int] | None = None, device="cpu",
              side: int | None = None) -> LightFieldCase:
    """Synthetic inputs of config `name`; `size` overrides H=W."""
    device = torch.device(device)
    name = name.lower()
    seed = {"c1": 1, "c2": 2, "c2b": 2, "c3": 3, "c4": 4, "c5": 5}[name]
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    rng = np.random.default_rng(seed)
    if isinstance(size, tuple):
        h, w = size
    elif size is not None:
        h = w = int(size)
    else:
        h = w = {"c1": 128, "c2": 512, "c2b": 1024, "c3": 1024, "c4": 2048}.get(name, 0)

    if name == "c1":
        sd = side or 5
        d = np.linspace(-1.5, 1.5, 12)
        tex, masks = _planes(gen, 12, 1, h, w, 2.0, device)
        coords = grid_coords(sd)
        views = _finish(_composite(tex, masks, d, coords), gen, 0.01)
        return LightFieldCase("c1", views, coords[:, 0], coords[:, 1], d, render_coords=coords)

    if name in ("c2", "c2b", "c4"):
        big = name == "c4"
        sd = side or (17 if big else 9)
        n = 64 if big else 30
        dmax = 6.0 if big else 3.0
        n_occ = 16 if big else 8
        d = np.linspace(-dmax, dmax, n)
        plane_d = np.concatenate(([-dmax], np.sort(rng.uniform(-dmax, dmax, n_occ))))
        tex, masks = _planes(gen, n_occ + 1, 3, h, w, 1.5, device)
        coords = grid_coords(sd)
        views = _finish(_composite(tex, masks, plane_d, coords, chunk=4 if big else 16), gen, 0.005)
        rc = np.concatenate([coords, coords + 0.5]) if not big else coords
        return LightFieldCase(name, views, coords[:, 0], coords[:, 1], d, render_coords=rc,
                              meta={"plane_d": plane_d})

    if name == "c3":
        raise ValueError("c3 needs a renderer: use harness.focal.make_focal_case")
    raise ValueError(f"unknown config {name!r}")


def random_fdl_layers(n: int, c: int, h: int, w: int, device="cpu", seed: int = 5,
                      dtype=torch.complex64) -> torch.Tensor:
    """C5 layers: rfft2 of i.i.d. U[0, 1/64] real images, (n, C, H, W//2+1)."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    out = torch.empty((n, c, h, w // 2 + 1), dtype=dtype, device=device)
    for k in range(n):
        img = torch.rand((c, h, w), generator=gen, dtype=torch.float32, device=device) / 64.0
        out[k] = torch.fft.rfft2(img.to(torch.float64)).to(dtype)
    return out


def render_requests_c5(count: int, seed: int = 5):
    """C5 requests: u,v ~ U[-4,4], s ~ U[-5,5], aperture radius r ~ U[0,3] -> f = 2r
    with one disk of diameter 1."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(-4, 4, count)
    v = rng.uniform(-4, 4, count)
    s = rng.uniform(-5, 5, count)
    r = rng.uniform(0, 3, count)
    return u, v, s, 2.0 * r

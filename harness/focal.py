"""C3 focal-stack inputs — harness, not product.

Ground truth: 48 fronto-parallel planes at d = linspace(-4, 4, 48) (texture
sigma 2 px, 30 % blob masks, full background at the farthest plane).  The GT
layers are the rfft2 of the visible central-view content of each plane (the
FDL definition).  The 40 focal images are renders of that
GT model at u = v = 0, s = f_i, f = 1 through a disk aperture of diameter 8
(the reference's `render`, render.py:228-248, restated here in torch float64
with the same separable bilinear aperture lookup, lfmodel.py:101-122).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .synth import LightFieldCase, _planes, grid_coords


def _axis_lookup(q, axis):
    step = axis[1] - axis[0]
    pos = (q - axis[0]) / step
    n = axis.numel()
    ok = (pos >= 0) & (pos <= n - 1)
    i0 = torch.clamp(torch.floor(pos), 0, n - 2).to(torch.long)
    fr = torch.clamp(pos - i0, 0.0, 1.0)
    return i0, fr, ok


def aperture_grid_torch(table, xi_x, xi_y, t, ox, oy):
    """psi_hat(t wx, t wy) on the (H, Whp) grid, float64, OOB -> 0."""
    iy, fy, oky = _axis_lookup(t * oy, xi_y)
    ix, fx, okx = _axis_lookup(t * ox, xi_x)
    rows = table[iy, :] * (1 - fy)[:, None] + table[iy + 1, :] * fy[:, None]
    out = rows[:, ix] * (1 - fx)[None, :] + rows[:, ix + 1] * fx[None, :]
    out = out * oky[:, None] * okx[None, :]
    return out


def make_focal_case(size: int | None = None, device="cpu", n_images: int = 40, n_layers: int = 48,
                    diameter: float = 8.0) -> LightFieldCase:
    from paper_1901_06919_b200.render import aperture_spectrum

    device = torch.device(device)
    h = w = int(size or 1024)
    gen = torch.Generator(device=device)
    gen.manual_seed(3)
    d = np.linspace(-4, 4, n_layers)
    tex, masks = _planes(gen, n_layers, 1, h, w, 2.0, device)
    # visible central-view content: plane k minus everything nearer (larger d) in front of it
    vis = torch.empty((n_layers, h, w), dtype=torch.float64, device=device)
    cover = torch.zeros((h, w), dtype=torch.float64, device=device)
    for k in range(n_layers - 1, -1, -1):
        vis[k] = tex[k, 0] * masks[k] * (1.0 - cover)
        cover = cover + masks[k] * (1.0 - cover)
    gt = torch.fft.rfft2(vis)  # (n, H, Whp)
    ap = aperture_spectrum("disk", diameter=diameter)
    table = torch.as_tensor(np.asarray(ap.table, dtype=np.float64), device=device)
    xi_x = torch.as_tensor(ap.xi_x, device=device)
    xi_y = torch.as_tensor(ap.xi_y, device=device)
    ox = torch.arange(w // 2 + 1, dtype=torch.float64, device=device) / w
    if w % 2 == 0:
        ox[-1] = -0.5
    oy = torch.fft.fftfreq(h, dtype=torch.float64, device=device)
    focus = np.linspace(-4, 4, n_images)
    imgs = torch.empty((n_images, h, w), dtype=torch.float64, device=device)
    for i, fi in enumerate(focus):
        acc = torch.zeros_like(gt[0])
        for k in range(n_layers):
            acc += gt[k] * aperture_grid_torch(table, xi_x, xi_y, float(fi - d[k]), ox, oy)
        imgs[i] = torch.fft.irfft2(acc, s=(h, w))
    views = imgs[..., None].to(torch.float32).contiguous()
    zeros = np.zeros(n_images)
    return LightFieldCase("c3", views, zeros, zeros.copy(), d, s=focus,
                          aperture={"shape": "disk", "diameter": diameter},
                          render_coords=grid_coords(9), meta={"gt_layers": gt})

"""CUDA-graph replay of a construction (+ renders) for a fixed acquisition geometry.

The latency-bound shapes (config 1: 25 views of 128 x 128, 0.24 ms of kernels
behind ~10 launches plus host planning per call) spend
more time in launch gaps and parameter staging than in kernels.  When the
geometry is fixed -- the same rig shooting frame after frame, the same set of
render requests -- everything but the pixel values is constant, so the whole
step is captured ONCE into a CUDA graph:

    K0 (pad + R2C + per-view sums) -> default lambda (device) -> K1 axis tables,
    solve, residual screen -> K2 -> [K3 + K4 for a fixed request list]

and replayed with new views copied into a static input buffer.  The C ABI
stages host parameter blocks through a reused pinned ring, which a graph must
not depend on: the capture runs inside a staging arena
(`fdl_staging_arena_begin`, include/fdl_b200.h) that gives every block its own
pinned allocation for the graph's lifetime.

What the graph does NOT do: the host-driven fallbacks.  `status` (per-bin
FDL_BIN_* flags) is left on the device; `check()` reads it (one
synchronisation) and raises if any bin broke down or is suspect -- rebuild that
frame with `construct_fdl`.  On the configs' well-posed inputs no bin is ever
flagged (tools/diag_screen.py).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .construct import (DEFAULT_EPS, _require_cuda, default_pad_margin, lambda_device, resolve_shifts, solve_slab,
                        symmetrize, views_to_spectra)
from .lfmodel import FdlModel, ShiftParams, ViewSet
from .render import render_many_device
from .spectra import FrequencyGrid

__all__ = ["GraphedConstruct"]


class GraphedConstruct:
    """construct_fdl (+ render_many) captured for one geometry; call it with new views.

    views_like: a ViewSet giving the geometry (u, v, apertures, shapes); its images seed
    the warm-up run.  requests: optional list of RenderRequest rendered inside the graph.
    """

    def __init__(self, views_like: ViewSet, shifts: ShiftParams, requests=None, lam: float | None = None,
                 eps: float = DEFAULT_EPS, pad_margin: int | None = None, device=None):
        torch = _require_cuda()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.meta, self.shifts, self.requests = views_like, shifts, list(requests or [])
        self.lam, self.eps = lam, float(eps)
        self.pu, self.pv, self.d = resolve_shifts(views_like, shifts)
        self.pad = default_pad_margin(self.pu, self.pv) if pad_margin is None else int(pad_margin)
        m, H, W, C = views_like.images.shape
        self.dims = (m, H, W, C)
        self.grid = FrequencyGrid(width=W + 2 * self.pad, height=H + 2 * self.pad)
        with torch.cuda.device(self.device):
            self.static_views = torch.empty((m, H, W, C), dtype=torch.float32, device=self.device)
            self._load(views_like.images)
            self._step()  # warm-up: cuFFT plans, constant tables, kernel attributes, allocator pools
            torch.cuda.synchronize(self.device)
            L = nat.lib()
            self._arena = L.fdl_staging_arena_begin()
            if not self._arena:
                raise nat.FdlNativeError("a staging arena is already open on this thread")
            self.graph = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
                    self.layers, self.status, self.lam_dev, self.images = self._step()
            finally:
                L.fdl_staging_arena_end(self._arena)
        self.model = FdlModel(disparities=self.d, layers=self.layers, grid=self.grid, width=W, height=H,
                              pad_margin=self.pad, color_space=views_like.color_space, calibration=shifts,
                              lambda_used=lam)

    def _load(self, images):
        import torch
        src = images if isinstance(images, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(images, np.float32))
        self.static_views.copy_(src.to(torch.float32), non_blocking=True)

    def _step(self):
        """One construction (+ renders) with no host synchronisation."""
        import torch
        m, H, W, C = self.dims
        Hp, Wp = self.grid.height, self.grid.width
        spectra, sumsq = views_to_spectra(self.static_views, self.pad)
        lam_dev = lambda_device(sumsq, self.grid.num_entries, m) if self.lam is None else None
        status = torch.zeros((Hp, Wp // 2 + 1), dtype=torch.int8, device=self.device)
        factored = self.shifts.is_factored  # (as construct_fdl: the fast paths key on the factored u, v)
        layers, _, _ = solve_slab(spectra, m, len(self.d), C, Hp, Wp, np.arange(Hp), self.pu, self.pv, self.d,
                                  self.lam, self.eps, views=self.meta, u=self.shifts.u if factored else None,
                                  v=self.shifts.v if factored else None, status=status, count=False, lam_dev=lam_dev)
        symmetrize(layers, Hp, Wp)
        images = None
        if self.requests:
            model = FdlModel(disparities=self.d, layers=layers, grid=self.grid, width=W, height=H,
                             pad_margin=self.pad, color_space=self.meta.color_space)
            images, _ = render_many_device(model, self.requests, batch=max(64, len(self.requests)))
        return layers, status, lam_dev, images

    def __call__(self, images=None):
        """Replay with new view data (None: the views already in `static_views`).  Returns
        (model, images): the resident model and the (V, H, W, C) float32 renders (or None);
        both are overwritten by the next replay."""
        import torch
        with torch.cuda.device(self.device):
            if images is not None:
                self._load(images)
            self.graph.replay()
        return self.model, self.images

    def check(self):
        """Synchronise and make sure no bin of the last replay needed a host-driven fallback."""
        flagged = int((self.status != 0).sum().item())
        if flagged:
            raise nat.FdlNativeError(f"{flagged} bins of the graphed construction need the fallback / residual "
                                     "audit: rebuild this frame with construct_fdl")
        if self.lam_dev is not None:
            self.model.lambda_used = float(self.lam_dev.item())
        return self.model

    def __del__(self):
        arena = getattr(self, "_arena", None)
        if arena:
            try:
                self.graph = None
                nat.lib().fdl_staging_arena_free(arena)
            except Exception:
                pass

"""Render-service backend on the GPU (the reference's
`RenderService.render_bytes`, serve.py:115-143).

The reference's HTTP front end (ThreadingHTTPServer, static viewer files) is out
of scope; what is rebuilt here is the part that sits on the
render hot path and that the front end calls from its worker threads:

    query string -> RenderRequest -> K3/K4 on the device
                 -> K6 quantisation to 8 bits ON THE DEVICE (fdl_images_to_u8)
                 -> one D2H copy of H*W*C BYTES (the reference moves no data but
                    converts H*W*C float64 on the host)
                 -> PNG / JPEG container on the host (Pillow, as the reference)

`RenderService` keeps the reference's constructor, `info`, `parse_query`,
`render_bytes`, error type and cache policy, so the reference's handler
(serve.py:146-195) can be pointed at it unchanged; `render_batch_bytes` is the
batched form (one K3/K4 launch set for many queries).  Identical queries give
byte-identical responses (the render is deterministic and results are cached
by the canonical query key, serve.py:116-121).
"""

from __future__ import annotations

import io as _io
import json
import math
import os
import threading
import time
from collections import OrderedDict
from urllib.parse import parse_qsl

import numpy as np

from . import _native as nat
from .lfmodel import FdlModel
from .render import RenderRequest, aperture_spectrum, render_many_device

__all__ = ["QueryError", "RenderService", "quantise_u8"]

CACHE_ENTRIES = 32  # serve.py:29


class QueryError(ValueError):
    """A client error with its HTTP status (serve.py:32-35)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def _number(params: dict, key: str, fallback: float) -> float:
    text = params.get(key)
    if text is None:
        return fallback
    try:
        value = float(text)
    except ValueError:
        raise QueryError(400, f"malformed parameter {key!r}: {text!r}") from None
    if not math.isfinite(value):
        raise QueryError(400, f"parameter {key!r} must be finite")
    return value


@nat.on_device(lambda images_dev: images_dev.device)
def quantise_u8(images_dev):
    """(…) float32 CUDA tensor -> uint8 CUDA tensor of the same shape:
    round_half_even(clip(x, 0, 1) * 255) in float64 on the device (serve.py:127)."""
    import torch
    src = images_dev.contiguous()
    out = torch.empty(src.shape, dtype=torch.uint8, device=src.device)
    nat.check(nat.lib().fdl_images_to_u8(src.data_ptr(), src.numel(), out.data_ptr(), nat.stream_handle(src.device)),
              "fdl_images_to_u8")
    return out


def _container(pixels: np.ndarray, fmt: str, jpeg_q: int) -> tuple[str, bytes]:
    from PIL import Image
    frame = Image.fromarray(pixels[..., 0] if pixels.shape[-1] == 1 else pixels)
    sink = _io.BytesIO()
    if fmt == "jpeg":
        frame.save(sink, format="JPEG", quality=jpeg_q)
        return "image/jpeg", sink.getvalue()
    frame.save(sink, format="PNG")
    return "image/png", sink.getvalue()


class RenderService:
    """Query parsing, GPU rendering and encoding around one immutable model (serve.py:51-143)."""

    def __init__(self, model: FdlModel, threads: int | None = None):
        self.model = model
        self.apertures = {  # one table per shape for the service's lifetime (serve.py:55-59)
            "pinhole": aperture_spectrum("pinhole"),
            "disk": aperture_spectrum("disk", diameter=1.0),
            "square": aperture_spectrum("square", side=1.0),
        }
        self._gate = threading.BoundedSemaphore(threads or os.cpu_count() or 1)
        self._cache: OrderedDict[str, tuple[str, bytes, float]] = OrderedDict()
        self._cache_lock = threading.Lock()
        model.layers_device()  # fail fast without a CUDA device / the native library

    def info(self) -> dict:
        m, cal = self.model, self.model.calibration
        hull = None
        if cal is not None and cal.is_factored:
            hull = {"u": [float(cal.u.min()), float(cal.u.max())], "v": [float(cal.v.min()), float(cal.v.max())]}
        return {"width": m.width, "height": m.height, "n": m.num_layers, "d": [float(x) for x in m.disparities],
                "hull": hull, "apertures": sorted(self.apertures), "color_space": m.color_space,
                "channels": m.channels}

    def parse_query(self, query: str):
        """(RenderRequest, "png" | "jpeg", jpeg quality); QueryError 400 / 422 as the reference (serve.py:86-113)."""
        params = dict(parse_qsl(query, keep_blank_values=True))
        u, v, s, f = (_number(params, k, 0.0) for k in ("u", "v", "s", "f"))
        if f < 0:
            raise QueryError(400, "parameter 'f' must be >= 0")
        shape = params.get("aperture", "disk")
        if shape not in self.apertures:
            raise QueryError(422, f"unknown aperture {shape!r}")
        quality = params.get("quality", "png")
        fmt, jpeg_q = "png", 85
        if quality.startswith("jpeg"):
            fmt = "jpeg"
            _, dash, level = quality.partition("-")
            if dash:
                try:
                    jpeg_q = int(level)
                except ValueError:
                    raise QueryError(400, f"malformed parameter 'quality': {quality!r}") from None
                if not 1 <= jpeg_q <= 100:
                    raise QueryError(400, "jpeg quality must be in 1..100")
        elif quality != "png":
            raise QueryError(400, f"malformed parameter 'quality': {quality!r}")
        return RenderRequest(u=u, v=v, s=s, f=f, aperture=self.apertures[shape]), fmt, jpeg_q

    @staticmethod
    def _key(query: str) -> str:
        return json.dumps(sorted(parse_qsl(query, keep_blank_values=True)))

    def _lookup(self, key):
        with self._cache_lock:
            hit = self._cache.get(key)
            if hit is not None:
                self._cache.move_to_end(key)
            return hit

    def _remember(self, key, value):
        with self._cache_lock:
            self._cache[key] = value
            while len(self._cache) > CACHE_ENTRIES:
                self._cache.popitem(last=False)

    def _pixels(self, reqs) -> np.ndarray:
        """(V, H, W, C) uint8 host pixels of the requests: render + quantise on the device, bytes over PCIe."""
        import torch
        imgs, _ = render_many_device(self.model, reqs)
        q = quantise_u8(imgs)
        host = torch.empty(q.shape, dtype=torch.uint8, pin_memory=True)
        host.copy_(q, non_blocking=True)
        torch.cuda.current_stream(q.device).synchronize()
        return host.numpy()

    def render_bytes(self, query: str) -> tuple[str, bytes, float]:
        """(content type, encoded image, render milliseconds) for one query string (serve.py:115-143)."""
        key = self._key(query)
        hit = self._lookup(key)
        if hit is not None:
            return hit
        req, fmt, jpeg_q = self.parse_query(query)
        t0 = time.perf_counter()
        with self._gate:
            pixels = self._pixels([req])[0]
        ms = (time.perf_counter() - t0) * 1000.0
        out = _container(pixels, fmt, jpeg_q) + (ms,)
        self._remember(key, out)
        return out

    def render_batch_bytes(self, queries) -> list[tuple[str, bytes, float]]:
        """`render_bytes` for many queries with ONE batched render of the uncached ones."""
        queries = list(queries)
        keys = [self._key(q) for q in queries]
        out = [self._lookup(k) for k in keys]
        todo = [i for i, hit in enumerate(out) if hit is None]
        if todo:
            parsed = [self.parse_query(queries[i]) for i in todo]
            t0 = time.perf_counter()
            with self._gate:
                pixels = self._pixels([p[0] for p in parsed])
            ms = (time.perf_counter() - t0) * 1000.0 / len(todo)
            for slot, i in enumerate(todo):
                out[i] = _container(pixels[slot], parsed[slot][1], parsed[slot][2]) + (ms,)
                self._remember(keys[i], out[i])
        return out

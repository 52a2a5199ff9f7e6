"""Golden fixtures of the pipelines (pipeline.py:140-219), FROM THE REFERENCE ITSELF.

    python tests/golden/make_pipeline.py     (build container only)

pipeline.npz: a 3 x 3 RGB two-layer light field (the reference's own
`synthesize_lightfield`, float32 inputs) and the reference's outputs of
interpolate_views (known shifts, and with calibration) and denoise (factored
known shifts, and relaxed refinement).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

import fdl  # noqa: E402  (the reference)
from fdl import CalibConfig, SceneSpec, ShiftParams, ViewSet  # noqa: E402
from fdl.pipeline import PipelineConfig, denoise, interpolate_views  # noqa: E402

from make_golden import quadrant_masks, smooth_texture  # noqa: E402


def main():
    rng = np.random.default_rng(77)
    h = w = 32
    scene = SceneSpec(masks=quadrant_masks(h, w, 2), disparities=[0.0, 1.0], texture=smooth_texture(rng, h, w))
    g = np.arange(3) - 1.0
    coords = np.array([(u, v) for v in g for u in g])
    base = fdl.synthesize_lightfield(scene, coords)
    gray = np.asarray(base.images)
    rgb = np.concatenate([gray, 0.8 * gray, 0.6 * gray + 0.1], axis=3)
    rgb = (rgb + 0.01 * rng.standard_normal(rgb.shape)).astype(np.float32)
    views = ViewSet(images=rgb, u=coords[:, 0], v=coords[:, 1])
    d = np.linspace(-0.5, 1.5, 6)
    known = ShiftParams.factored(coords[:, 0], coords[:, 1], d)
    targets = np.array([[0.5, 0.5], [-0.5, 0.25], [1.5, 0.0]])
    out = {"images": rgb, "coords": coords, "d": d, "targets": targets}
    sink = {}
    iv = interpolate_views(views, targets, PipelineConfig(known_shifts=known), report_sink=sink)
    out["interp_known"] = iv.images
    out["interp_flags"] = np.array(sink["extrapolated"])
    cal = CalibConfig(n_layers=2, batch_size=10**6, grid_dims=(3, 3), d_min=-0.2, d_max=1.2, max_iters=30,
                      seed=0, lam=1e-4)
    out["interp_calib"] = interpolate_views(views, targets, PipelineConfig(calib=cal)).images
    dn, rep = denoise(views, PipelineConfig(known_shifts=known))
    out["denoise_known"] = dn.images
    out["denoise_known_psnr"] = np.array(rep.per_view_psnr)
    cal_r = CalibConfig(n_layers=6, batch_size=10**6, max_iters=8, seed=0, lam=1e-4)
    dr, rep_r = denoise(views, PipelineConfig(known_shifts=known, calib=cal_r), relaxed=True)
    out["denoise_relaxed"] = dr.images
    out["denoise_relaxed_psnr"] = np.array(rep_r.per_view_psnr)
    np.savez_compressed(HERE / "pipeline.npz", **out)
    print({k: np.shape(v) for k, v in out.items()}, rep.mean_psnr, rep_r.mean_psnr)


if __name__ == "__main__":
    main()

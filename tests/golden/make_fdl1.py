"""FDL1 model files written BY THE REFERENCE (fdl/io.py:157-180), for the
format-compatibility tests of paper_1901_06919_b200/io.py.  Run in the build
container (the reference is importable from /root/reference/pkg/src):

    python tests/golden/make_fdl1.py

Writes ref_factored.fdl (factored calibration block, pad 1) and
ref_relaxed.fdl (relaxed block, gamma model, lambda = NaN sentinel absent).
The scene is the reference's own tests' small model (test_io.py:120-128).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from fdl import SceneSpec, ShiftParams, construct_fdl, synthesize_lightfield  # noqa: E402
from fdl.io import save_model  # noqa: E402

sys.path.insert(0, str(HERE))
from make_golden import grid_coords, quadrant_masks, smooth_texture  # noqa: E402


def main():
    rng = np.random.default_rng(1901)
    scene = SceneSpec(masks=quadrant_masks(16, 16, 2), disparities=[0.0, 1.0],
                      texture=smooth_texture(rng, 16, 16))
    views = synthesize_lightfield(scene, grid_coords(3))
    shifts = ShiftParams.factored(views.u, views.v, [0.0, 1.0])
    model = construct_fdl(views, shifts, lam=1e-4, pad_margin=1)
    save_model(HERE / "ref_factored.fdl", model)
    pu = np.outer(np.arange(9) - 4.0, model.disparities)
    model.calibration = ShiftParams.relaxed(pu, pu * 0.5, d=model.disparities)
    model.lambda_used = None
    save_model(HERE / "ref_relaxed.fdl", model)
    print("wrote", HERE / "ref_factored.fdl", HERE / "ref_relaxed.fdl")


if __name__ == "__main__":
    main()

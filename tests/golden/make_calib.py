"""Golden fixtures of the calibration path, generated FROM THE REFERENCE ITSELF.

    python tests/golden/make_calib.py      (build container; the reference is
                                            importable from /root/reference/pkg/src)

calib.npz holds float32 view stacks (two-layer occluded scenes built by the
reference's own `synthesize_lightfield` from the reference tests' fixtures,
tests/conftest.py restated in make_golden.py) and the reference's outputs:
objective / layer coefficients / shift-matrix gradients / data residual at
perturbed parameters (calibrate.py:197-259), a full-batch and a stochastic
`calibrate` run (:411-439) and a `calibrate_relaxed` refinement (:442-459).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

import fdl  # noqa: E402  (the reference)
from fdl import CalibConfig, SceneSpec, ShiftParams, ViewSet, calibrate, calibrate_relaxed  # noqa: E402
from fdl.calibrate import data_residual, frequency_pool, grad_shift_matrix, layer_coefficients, objective  # noqa: E402
from fdl.spectra import FrequencyGrid  # noqa: E402

from make_golden import quadrant_masks, smooth_texture  # noqa: E402


def grid3():
    g = np.arange(3) - 1.0
    return np.array([(u, v) for v in g for u in g])


def two_layer(rng, h, w, jitter):
    scene = SceneSpec(masks=quadrant_masks(h, w, 2), disparities=[0.0, 1.0], texture=smooth_texture(rng, h, w))
    coords = grid3() + jitter * rng.uniform(-1, 1, (9, 2))
    coords -= coords.mean(axis=0, keepdims=True)
    views = fdl.synthesize_lightfield(scene, coords)
    imgs = np.asarray(views.images, dtype=np.float32)  # float32 inputs: both sides upcast the same values
    return ViewSet(images=imgs, u=coords[:, 0], v=coords[:, 1]), coords


def main():
    rng = np.random.default_rng(2024)
    out = {}
    # A: batch quantities at perturbed parameters (32 x 32, three layers, RGB)
    va, ca = two_layer(rng, 32, 32, 0.15)
    rgb = np.repeat(np.asarray(va.images), 3, axis=3) * np.array([1.0, 0.8, 0.6], np.float32)
    va = ViewSet(images=rgb.astype(np.float32), u=va.u, v=va.v)
    u = ca[:, 0] + 0.05 * rng.standard_normal(9)
    v = ca[:, 1] + 0.05 * rng.standard_normal(9)
    d = np.array([-0.3, 0.4, 1.1])
    grid = FrequencyGrid(width=32, height=32)
    sub = rng.permutation(frequency_pool(grid))[:200]
    sh = ShiftParams.factored(u, v, d)
    out.update(A_images=va.images, A_u=u, A_v=v, A_d=d, A_sub=sub.astype(np.int64))
    out["A_obj_pool_layer"] = objective(va, u, v, d, lam=1e-3)
    out["A_obj_sub_identity"] = objective(va, u, v, d, lam=1e-2, freq_indices=sub, reg_kind="identity")
    out["A_obj_sub_lam0"] = objective(va, u, v, d, lam=0.0, freq_indices=sub)
    x = layer_coefficients(va, sh, lam=1e-3, freq_indices=sub)
    out["A_x_sub"] = x
    gpu, gpv = grad_shift_matrix(va, sh, x, freq_indices=sub, lam=1e-3)
    out["A_gpu_sub"], out["A_gpv_sub"] = gpu, gpv
    out["A_resid_pool"] = data_residual(va, sh, lam=1e-3)
    # B: full-batch calibration, 48 x 48 grayscale
    vb, cb = two_layer(rng, 48, 48, 0.15)
    cfg = CalibConfig(n_layers=2, batch_size=10**6, grid_dims=(3, 3), d_min=-0.2, d_max=1.2, max_iters=40,
                      seed=0, lam=1e-4)
    res = calibrate(vb, cfg)
    out.update(B_images=vb.images, B_coords=cb, B_u=res.u, B_v=res.v, B_d=res.d,
               B_hist=np.array([h.objective for h in res.history]), B_converged=res.converged)
    # C: stochastic batches (256 of the pool), layer regulariser, three layers
    cfg_c = CalibConfig(n_layers=3, batch_size=256, grid_dims=(3, 3), d_min=-0.5, d_max=1.5, max_iters=25, seed=3,
                        lam=1e-3)
    res_c = calibrate(vb, cfg_c)
    out.update(C_u=res_c.u, C_v=res_c.v, C_d=res_c.d, C_hist=np.array([h.objective for h in res_c.history]))
    # D: relaxed refinement of B
    cfg_d = CalibConfig(n_layers=2, batch_size=10**6, max_iters=15, seed=0, lam=1e-4)
    rel, hist = calibrate_relaxed(vb, res.shift_params, cfg_d)
    out.update(D_pu=rel.pu, D_pv=rel.pv, D_hist=np.array([h.objective for h in hist]))
    np.savez_compressed(HERE / "calib.npz", **out)
    print({k: (np.shape(v_) if np.ndim(v_) else v_) for k, v_ in out.items() if not k.endswith("images")})


if __name__ == "__main__":
    main()

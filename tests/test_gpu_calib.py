"""Calibration on the GPU (paper_1901_06919_b200.calibrate, csrc/k5_calib.cu)
against the reference's outputs (tests/golden/calib.npz) and the oracle.

Batch quantities (objective, layer coefficients, gradients) are fp64 on both
sides: they agree to ~1e-12 relative (Cholesky vs the reference's LU, cuFFT
vs pocketfft); gates 1e-8.  Descent runs compare the accepted iterates; the
gates allow for an accept/reject decision that rounding could flip."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cal():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import importlib
    return importlib.import_module("paper_1901_06919_b200.calibrate")  # the module (the package exports the function)


@pytest.fixture(scope="module")
def g():
    return load_golden("calib")


def views_a(g):
    from paper_1901_06919_b200 import ViewSet
    return ViewSet(images=g["A_images"], u=g["A_u"], v=g["A_v"])


def test_objective_matches_reference(cal, g):
    va = views_a(g)
    u, v, d = g["A_u"], g["A_v"], g["A_d"]
    assert cal.objective(va, u, v, d, lam=1e-3) == pytest.approx(float(g["A_obj_pool_layer"]), rel=1e-9)
    assert cal.objective(va, u, v, d, lam=1e-2, freq_indices=g["A_sub"], reg_kind="identity") == pytest.approx(
        float(g["A_obj_sub_identity"]), rel=1e-9)
    assert cal.objective(va, u, v, d, lam=0.0, freq_indices=g["A_sub"]) == pytest.approx(
        float(g["A_obj_sub_lam0"]), rel=1e-9)


def test_layers_gradients_residual_match_reference(cal, g):
    from paper_1901_06919_b200 import ShiftParams
    va = views_a(g)
    sh = ShiftParams.factored(g["A_u"], g["A_v"], g["A_d"])
    x = cal.layer_coefficients(va, sh, lam=1e-3, freq_indices=g["A_sub"])
    np.testing.assert_allclose(x, g["A_x_sub"], rtol=1e-8, atol=1e-10 * np.abs(g["A_x_sub"]).max())
    gpu, gpv = cal.grad_shift_matrix(va, sh, g["A_x_sub"], freq_indices=g["A_sub"], lam=1e-3)
    np.testing.assert_allclose(gpu, g["A_gpu_sub"], rtol=1e-8, atol=1e-10 * np.abs(g["A_gpu_sub"]).max())
    np.testing.assert_allclose(gpv, g["A_gpv_sub"], rtol=1e-8, atol=1e-10 * np.abs(g["A_gpv_sub"]).max())
    assert cal.data_residual(va, sh, lam=1e-3) == pytest.approx(float(g["A_resid_pool"]), rel=1e-9)


def test_gradients_match_oracle_on_random_parameters(cal, rng):
    from oracle import fdl_oracle as O
    from paper_1901_06919_b200 import ShiftParams, ViewSet
    m, n, h, w = 6, 4, 24, 30
    imgs = rng.uniform(0, 1, (m, h, w, 1)).astype(np.float32)
    pu, pv = rng.normal(size=(m, n)), rng.normal(size=(m, n))
    views = ViewSet(images=imgs, u=np.zeros(m), v=np.zeros(m))
    sh = ShiftParams.relaxed(pu, pv, d=np.linspace(-1, 1, n))
    spec = O.luma_spectra(imgs)
    pool = O.frequency_pool(w, h)
    val, x, (gu, gv) = O.calib_batch(pu, pv, spec, pool, w, h, 1e-3, O.layer_regularizer(n), grad=True)
    xg = cal.layer_coefficients(views, sh, lam=1e-3)
    np.testing.assert_allclose(xg, x, rtol=1e-8, atol=1e-10 * np.abs(x).max())
    gpu, gpv = cal.grad_shift_matrix(views, sh, x, lam=1e-3)
    np.testing.assert_allclose(gpu, gu, rtol=1e-8, atol=1e-10 * np.abs(gu).max())
    np.testing.assert_allclose(gpv, gv, rtol=1e-8, atol=1e-10 * np.abs(gv).max())


def test_full_batch_calibration_matches_reference(cal, g):
    from paper_1901_06919_b200 import ViewSet
    vb = ViewSet(images=g["B_images"], u=np.zeros(9), v=np.zeros(9))
    cfg = cal.CalibConfig(n_layers=2, batch_size=10**6, grid_dims=(3, 3), d_min=-0.2, d_max=1.2, max_iters=40,
                          seed=0, lam=1e-4)
    res = cal.calibrate(vb, cfg)
    hist = np.array([h.objective for h in res.history])
    k = min(len(hist), len(g["B_hist"]))
    np.testing.assert_allclose(hist[:k], g["B_hist"][:k], rtol=1e-6)
    np.testing.assert_allclose(res.u, g["B_u"], atol=1e-6)
    np.testing.assert_allclose(res.v, g["B_v"], atol=1e-6)
    np.testing.assert_allclose(res.d, g["B_d"], atol=1e-6)
    assert np.all(np.diff(res.d) > 0) and abs(res.u.mean()) < 1e-9 and abs(res.v.mean()) < 1e-9


def test_stochastic_calibration_matches_reference(cal, g):
    from paper_1901_06919_b200 import ViewSet
    vb = ViewSet(images=g["B_images"], u=np.zeros(9), v=np.zeros(9))
    cfg = cal.CalibConfig(n_layers=3, batch_size=256, grid_dims=(3, 3), d_min=-0.5, d_max=1.5, max_iters=25,
                          seed=3, lam=1e-3)
    res = cal.calibrate(vb, cfg)
    hist = np.array([h.objective for h in res.history])
    k = min(len(hist), len(g["C_hist"]))
    np.testing.assert_allclose(hist[:k], g["C_hist"][:k], rtol=1e-6)
    np.testing.assert_allclose(res.d, g["C_d"], atol=1e-6)


def test_relaxed_refinement_matches_reference(cal, g):
    from paper_1901_06919_b200 import ShiftParams, ViewSet
    vb = ViewSet(images=g["B_images"], u=np.zeros(9), v=np.zeros(9))
    p0 = ShiftParams.factored(g["B_u"], g["B_v"], g["B_d"])
    cfg = cal.CalibConfig(n_layers=2, batch_size=10**6, max_iters=15, seed=0, lam=1e-4)
    rel, hist = cal.calibrate_relaxed(vb, p0, cfg)
    np.testing.assert_allclose([h.objective for h in hist][: len(g["D_hist"])], g["D_hist"][: len(hist)], rtol=1e-6)
    np.testing.assert_allclose(rel.pu, g["D_pu"], atol=1e-6)
    np.testing.assert_allclose(rel.pv, g["D_pv"], atol=1e-6)


def test_recovers_jittered_grid(cal, g):
    # the reference's test_recovers_jittered_grid (tests/test_calibrate.py:201-213) on the golden scene
    from paper_1901_06919_b200 import ViewSet
    vb = ViewSet(images=g["B_images"], u=np.zeros(9), v=np.zeros(9))
    cfg = cal.CalibConfig(n_layers=2, batch_size=10**6, grid_dims=(3, 3), d_min=-0.2, d_max=1.2, max_iters=2000,
                          seed=0, lam=1e-4)
    res = cal.calibrate(vb, cfg)
    pu, pv = res.shift_params.expand()
    coords = g["B_coords"]
    err = max(np.max(np.abs(pu - np.outer(coords[:, 0], [0.0, 1.0]))),
              np.max(np.abs(pv - np.outer(coords[:, 1], [0.0, 1.0]))))
    assert err < 1e-2
    objs = [h.objective for h in res.history]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(objs, objs[1:]))


def test_refuses_wide_aperture(cal):
    # tests/test_calibrate.py:72-78
    from paper_1901_06919_b200 import ViewSet, aperture_spectrum
    views = ViewSet(images=np.zeros((1, 8, 8, 1)), u=[0.0], v=[0.0],
                    apertures=[aperture_spectrum("disk", diameter=1.0)])
    with pytest.raises(ValueError, match="pinhole"):
        cal.objective(views, [0.0], [0.0], [0.0], lam=0.0)


def test_lstsq_minnorm_matches_numpy(rng):
    import ctypes
    import torch
    from paper_1901_06919_b200 import _native as nat
    B, n = 5, 6
    A = rng.normal(size=(B, n, 3)) + 1j * rng.normal(size=(B, n, 3))
    A = A @ A.conj().transpose(0, 2, 1)  # rank 3 of 6: exactly singular Hermitian
    b = rng.normal(size=(B, n, 1)) + 1j * rng.normal(size=(B, n, 1))
    At, bt = torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda()
    x = torch.empty((B, n, 1), dtype=torch.complex128, device="cuda")
    st = torch.zeros(B, dtype=torch.int8, device="cuda")
    L = nat.lib()
    ws = nat.workspace(L.fdl_lstsq_minnorm_workspace(B, n, n, 1), "cuda")
    nat.check(L.fdl_lstsq_minnorm(B, n, n, 1, At.data_ptr(), bt.data_ptr(), x.data_ptr(), st.data_ptr(),
                                  ws.data_ptr(), ws.numel(), nat.stream_handle()), "fdl_lstsq_minnorm")
    ref = np.stack([np.linalg.lstsq(A[i], b[i], rcond=None)[0] for i in range(B)])
    np.testing.assert_allclose(x.cpu().numpy(), ref, rtol=1e-8, atol=1e-10 * np.abs(ref).max())
    assert np.all(st.cpu().numpy() == 2)  # 2: minimum-norm solution (fdl_b200.h)

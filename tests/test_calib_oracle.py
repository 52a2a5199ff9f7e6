"""The calibration oracle (oracle/fdl_oracle.py: calib_batch & co.) against the
reference's own outputs (tests/golden/calib.npz, tests/golden/make_calib.py).
CPU only."""

import numpy as np

from conftest import load_golden
from oracle import fdl_oracle as O


def _batch(g, lam, bins=None, reg="layer", grad=False):
    imgs = g["A_images"]
    _, h, w, _ = imgs.shape
    spec = O.luma_spectra(imgs)
    bins = O.frequency_pool(w, h) if bins is None else bins
    n = len(g["A_d"])
    gamma = O.layer_regularizer(n) if reg == "layer" else np.eye(n)
    return O.calib_batch(np.outer(g["A_u"], g["A_d"]), np.outer(g["A_v"], g["A_d"]), spec, bins, w, h, lam, gamma,
                         grad=grad)


def test_oracle_objective_matches_reference():
    g = load_golden("calib")
    assert np.isclose(_batch(g, 1e-3)[0], g["A_obj_pool_layer"], rtol=1e-12)
    assert np.isclose(_batch(g, 1e-2, g["A_sub"], "identity")[0], g["A_obj_sub_identity"], rtol=1e-12)
    assert np.isclose(_batch(g, 0.0, g["A_sub"])[0], g["A_obj_sub_lam0"], rtol=1e-12)


def test_oracle_layers_and_gradients_match_reference():
    g = load_golden("calib")
    _, x, (gpu, gpv) = _batch(g, 1e-3, g["A_sub"], grad=True)
    np.testing.assert_allclose(x, g["A_x_sub"], rtol=1e-10, atol=1e-12 * np.abs(g["A_x_sub"]).max())
    np.testing.assert_allclose(gpu, g["A_gpu_sub"], rtol=1e-9, atol=1e-12 * np.abs(g["A_gpu_sub"]).max())
    np.testing.assert_allclose(gpv, g["A_gpv_sub"], rtol=1e-9, atol=1e-12 * np.abs(g["A_gpv_sub"]).max())


def test_oracle_regularizer_and_pool():
    gm = O.layer_regularizer(4)
    assert np.array_equal(np.diag(gm), [-2.0] * 4) and gm[0, 1] == 1.0 and gm[0, 2] == 0.0
    pool = O.frequency_pool(8, 6)
    wh = 5
    assert not np.any(pool % wh == 4) and not np.any(pool // wh == 3)
    assert len(pool) == 5 * 4

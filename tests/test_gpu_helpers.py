"""Per-bin public helpers and the minimum-norm fallback, on the GPU.

Mirrors the reference's own unit tests of these functions
(tests/test_construct.py:30-105 in the reference package): closed-form system
rows, scalar / ridge / dense-inverse solves, rank deficiency at lam = 0 and
the minimum-norm fallback for a degenerate system; plus a whole construction
whose DC bin is exactly singular (eps = 0) checked against the oracle, which
runs the reference's own fallback (construct.py:157-165, 205-210).
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fdl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_06919_b200 as pkg
    return pkg


def pinhole_views(fdl, m=2, h=8, w=8, u=None, v=None):
    return fdl.ViewSet(images=np.zeros((m, h, w, 1)), u=u if u is not None else np.zeros(m),
                       v=v if v is not None else np.zeros(m))


def test_system_row_phase(fdl):
    views = pinhole_views(fdl, 1, u=[0.5], v=[0.0])
    row = fdl.build_system_row(views, 0, (0.25, 0.0), [1.0])
    assert row[0] == pytest.approx(np.exp(1j * np.pi / 4), abs=1e-12)


def test_system_row_dc_is_ones(fdl):
    views = pinhole_views(fdl, 1, u=[1.3], v=[-0.4])
    views.apertures[0] = fdl.aperture_spectrum("disk", diameter=1.0)
    views.s[0] = 0.7
    row = fdl.build_system_row(views, 0, (0.0, 0.0), [-1.0, 0.5, 2.0])
    assert np.allclose(row, 1.0, atol=1e-9)


def test_scalar_and_ridge(fdl):
    x = fdl.solve_frequency(np.array([[2.0]]), np.array([4.0]), np.array([0.0]), 0.0)
    assert x[0] == pytest.approx(2.0, abs=1e-12)
    x = fdl.solve_frequency(np.array([[1.0]]), np.array([1.0]), np.array([1.0]), 1.0)
    assert x[0] == pytest.approx(0.5, abs=1e-12)


def test_matches_dense_inverse_oracle(fdl, rng):
    for _ in range(5):
        m, n = 6, 4
        A = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        b = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        reg = rng.uniform(0.5, 2.0, n)
        x = fdl.solve_frequency(A, b, reg, 1e-3)
        oracle = np.linalg.inv(A.conj().T @ A + 1e-3 * np.diag(reg)) @ (A.conj().T @ b)
        assert np.max(np.abs(x - oracle)) < 1e-10


def test_full_matrix_regularizer(fdl, rng):
    A = rng.standard_normal((3, 2)) + 1j * rng.standard_normal((3, 2))
    b = rng.standard_normal(3) + 1j * rng.standard_normal(3)
    R = np.array([[2.0, -1.0], [-1.0, 2.0]])
    x = fdl.solve_frequency(A, b, R, 0.5)
    oracle = np.linalg.solve(A.conj().T @ A + 0.5 * R, A.conj().T @ b)
    assert np.max(np.abs(x - oracle)) < 1e-10


def test_rank_deficiency_at_lambda_zero(fdl):
    with pytest.raises(fdl.RankDeficiencyError):
        fdl.solve_frequency(np.ones((2, 2), dtype=complex), np.ones(2, dtype=complex), np.ones(2), 0.0)
    with pytest.raises(fdl.RankDeficiencyError, match="ill-posed"):
        fdl.solve_frequency(np.ones((1, 3), dtype=complex), np.ones(1, dtype=complex), np.ones(3), 0.0)


def test_degenerate_falls_back_to_min_norm(fdl):
    A = np.ones((3, 2), dtype=complex)
    b = np.full(3, 2.0, dtype=complex)
    x = fdl.solve_frequency(A, b, np.full(2, 1e-18), 1e-12)
    assert np.all(np.isfinite(x))
    assert np.max(np.abs(A @ x - b)) < 1e-8
    assert abs(x[0] - x[1]) < 1e-6


def test_min_norm_matches_lstsq_on_random_degenerate(fdl, rng):
    # rank-deficient A (duplicated columns), vanishing regulariser: min-norm branch
    for _ in range(3):
        base = rng.standard_normal((5, 2)) + 1j * rng.standard_normal((5, 2))
        A = np.concatenate([base, base[:, :1]], axis=1)
        b = rng.standard_normal(5) + 1j * rng.standard_normal(5)
        reg = np.array([0.0, 1e-20, 0.0])
        x = fdl.solve_frequency(A, b, reg, 1e-14)
        w = np.sqrt(1e-14 * reg)
        ref = np.linalg.lstsq(np.vstack([A, np.diag(w)]), np.concatenate([b, np.zeros(3)]), rcond=None)[0]
        assert np.max(np.abs(x - ref)) < 1e-8 * max(1.0, np.max(np.abs(ref)))


def test_construct_singular_dc_bin_uses_fallback(fdl, rng):
    # two views at the same position, layers at d = 0 and 1, eps = 0: the DC bin's
    # normal matrix is exactly singular; the reference re-solves it by min-norm LS
    from oracle import fdl_oracle as O
    img = rng.uniform(0, 1, (2, 16, 16, 1))
    views = fdl.ViewSet(images=img, u=[0.0, 0.0], v=[0.0, 0.0])
    sh = fdl.ShiftParams.factored([0.0, 0.0], [0.0, 0.0], [0.0, 1.0])
    model = fdl.construct_fdl(views, sh, lam=1e-3, eps=0.0, pad_margin=0)
    assert fdl.last_construct_stats().fallback_bins >= 1
    ref = O.construct(img, np.zeros((2, 2)), np.zeros((2, 2)), np.array([0.0, 1.0]), lam=1e-3, eps=0.0, pad=0)
    assert rel_l2(model.layers, ref["layers"]) < 1e-6

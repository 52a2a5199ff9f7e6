"""Golden fixtures for the reference's normal-equation fallback
(construct.py:198-210), made by the reference itself.

Three mirror-symmetric views (u = -1, 0, 1; v = 0) and four layers
(d = -1.5 .. 1.5): rank(A^H A) <= 3 < 4 at every bin, so the regulariser alone
makes the normal matrices invertible.
  nearsingular : eps = 0, lam = 1e-12, 14 px -- the DC bin's matrix is exactly
                 singular, np.linalg.solve raises for the chunk and the
                 reference re-solves EVERY bin of it by minimum-norm LS;
  illcond      : eps = 1e-9, lam = 1e-6, 40 px -- cond(G) up to ~1e16, yet the
                 LU residuals stay <= ~1e-13 relative and nothing is re-solved.
  residfire    : four views, disparities (0, 1e-4, 1), eps = 1, lam = 5e-16, 12 px --
                 every normal matrix is positive definite (Cholesky succeeds on all
                 bins, np.linalg.solve does not raise) yet ONE bin's LU residual is
                 1.4e-8 > 1e-8 and the reference re-solves exactly that bin (found by
                 a parameter scan; the case VERDICT r1 asked for).
(`flagged` = the bins the reference's own test re-solved.)  Run here (the
reference is importable in the build container):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_nearsingular.py
"""

from pathlib import Path

import numpy as np

import fdl
from fdl import FrequencyGrid, ShiftParams, ViewSet, construct_fdl

HERE = Path(__file__).resolve().parent


def main():
    for name, size, lam, eps in (("nearsingular", 14, 1e-12, 0.0), ("illcond", 40, 1e-6, 1e-9)):
        case(name, size, lam, eps)
    case("residfire", 12, 5e-16, 1.0, seed=2, u=np.array([-1.0, 0.0, 1.0, 0.5]), v=np.array([0.0, 1.0, -1.0, 0.25]),
         d=np.array([0.0, 1e-4, 1.0]), f64_views=True)


def case(name, size, lam, eps, seed=2026, u=None, v=None, d=None, f64_views=False):
    rng = np.random.default_rng(seed)
    if u is None:
        u = np.array([-1.0, 0.0, 1.0])
        v = np.zeros(3)
        d = np.array([-1.5, -0.5, 0.5, 1.5])
    views = rng.uniform(0.0, 1.0, (len(u), size, size, 1))
    if not f64_views:
        views = views.astype(np.float32)
    vs = ViewSet(images=views.astype(np.float64), u=u, v=v)
    sh = ShiftParams.factored(u, v, d)
    model = construct_fdl(vs, sh, lam=lam, eps=eps)
    pad = model.pad_margin
    # which bins the reference re-solved: _solve_chunk's own test, replayed on its own normal equations
    pu, pv = np.outer(u, d), np.outer(v, d)
    img = np.pad(vs.images, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    hp, wp = img.shape[1:3]
    whp = wp // 2 + 1
    spec = np.fft.rfft2(np.moveaxis(img, 3, 1), axes=(-2, -1))
    b_all = spec.reshape(len(u), 1, hp * whp).transpose(2, 0, 1)
    grid = FrequencyGrid(wp, hp)
    q = np.arange(hp * whp)
    kx, ky = q % whp, q // whp
    px, py = fdl.construct._phase_tables(pu, pv, grid)
    A = fdl.construct._system_chunk(pu, pv, px, py, vs, d, grid, kx, ky)
    reg = (grid.omega_x[kx] ** 2 + grid.omega_y[ky] ** 2)[:, None] ** 2 * d[None, :] ** 4 + eps
    AH = A.conj().transpose(0, 2, 1)
    G = AH @ A
    G[:, np.arange(len(d)), np.arange(len(d))] += lam * reg
    rhs = AH @ b_all
    flagged = np.zeros(len(q), bool)
    res = np.full(len(q), np.nan)
    try:
        x = np.linalg.solve(G, rhs)
        flagged |= ~np.all(np.isfinite(x), axis=(1, 2))
        res = np.linalg.norm(G @ x - rhs, axis=(1, 2)) / np.maximum(np.linalg.norm(rhs, axis=(1, 2)),
                                                                     np.finfo(float).tiny)
        flagged |= res > 1e-8
    except np.linalg.LinAlgError:
        flagged[:] = True
    print(f"{name}: {hp}x{wp} grid, {int(flagged.sum())} of {len(q)} bins re-solved by the reference, "
          f"max cond {np.max(np.linalg.cond(G)):.2e}, max LU residual {np.nanmax(res) if np.isfinite(res).any() else np.nan:.2e}")
    np.savez_compressed(HERE / f"{name}.npz", views=views, u=u, v=v, d=d, lam=np.array(lam), eps=np.array(eps),
                        pad=np.array(pad), layers=model.layers, flagged=flagged, lu_residual=res)


if __name__ == "__main__":
    main()

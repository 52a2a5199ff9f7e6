"""Generate the golden fixtures of tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (the reference is importable from
/root/reference/pkg/src; it does not exist on the GPU box):

    python tests/golden/make_golden.py

Each fixture stores the float32 inputs, the reference's outputs (complex128
layers, lambda, float64 renders, render stats) and the parameters, so the
oracle (oracle/fdl_oracle.py) and the CUDA path can be checked against the
reference without it.  Inputs come from harness/ (seeded synthetic light
fields) or the reference's own test fixtures
(tests/conftest.py:7-52 restated: smooth_texture, quadrant_masks).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import fdl  # noqa: E402  (the reference)
from fdl import (FdlModel, RenderRequest, SceneSpec, ShiftParams, ViewSet,  # noqa: E402
                 aperture_spectrum, construct_fdl, last_render_stats, render, render_views_with_shifts,
                 synthesize_lightfield)
from fdl.spectra import FrequencyGrid  # noqa: E402

from harness.synth import grid_coords, make_case, random_fdl_layers, render_requests_c5  # noqa: E402


def smooth_texture(rng, h, w, cutoff=0.02):
    tex = rng.uniform(0, 1, (h, w))
    fx = np.fft.rfftfreq(w)
    fy = np.fft.fftfreq(h)
    lp = 1.0 / (1.0 + (fx[None, :] ** 2 + fy[:, None] ** 2) / cutoff)
    tex = np.fft.irfft2(np.fft.rfft2(tex) * lp, s=(h, w))
    return (tex - tex.min()) / np.ptp(tex)


def quadrant_masks(h, w, k):
    labels = np.zeros((h, w), int)
    if k > 1:
        labels[:, w // 2:] = 1
    if k > 2:
        labels[h // 2:, : w // 2] = 2
    if k > 3:
        labels[: h // 4, : w // 4] = 3
    return np.stack([labels == i for i in range(k)])


def ap_fields(prefix, ap):
    if ap is None or ap.is_pinhole:
        return {}
    return {f"{prefix}_table": ap.table, f"{prefix}_xi_x": ap.xi_x, f"{prefix}_xi_y": ap.xi_y}


def save(name, **arrays):
    path = HERE / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"{path.name}: {path.stat().st_size / 1e6:.2f} MB")


def floors(views, pu, pv, d, lam, pad, aps=None, s=None, bins=None):
    """The reference's own fp64 noise floor on these normal equations:
    relative L2 between its LU solution and (a) Cholesky, (b) LU with the layer
    order reversed, (c) LU with the phases of A evaluated exactly (long-double
    argument and sin/cos, i.e. an equally valid fp64 A differing by < 1 ulp)."""
    import scipy.linalg as sla
    m, n = pu.shape
    vs = ViewSet(images=views.astype(np.float64), u=np.zeros(m), v=np.zeros(m), s=s, apertures=aps)
    img = np.pad(vs.images, ((0, 0), (pad, pad), (pad, pad), (0, 0))) if pad else vs.images
    hp, wp = img.shape[1:3]
    whp = wp // 2 + 1
    spec = np.fft.rfft2(np.moveaxis(img, 3, 1), axes=(-2, -1))
    b_all = spec.reshape(m, img.shape[3], hp * whp).transpose(2, 0, 1)
    grid = FrequencyGrid(wp, hp)
    q = np.arange(hp * whp) if bins is None else bins
    kx, ky = q % whp, q // whp
    px, py = fdl.construct._phase_tables(pu, pv, grid)
    A = fdl.construct._system_chunk(pu, pv, px, py, vs, d, grid, kx, ky)
    # exact-phase A: long-double arguments
    L2 = np.longdouble
    twopi = 2 * np.pi * L2(1)
    twopi = L2("6.283185307179586476925286766559")
    ex = lambda P, om: (np.cos(twopi * P.astype(L2) * L2(1) * om.astype(L2)) + 1j * np.sin(twopi * P.astype(L2) * om.astype(L2))).astype(np.complex128)
    pxe = ex(pu[:, :, None], grid.omega_x[None, None, :])
    pye = ex(pv[:, :, None], grid.omega_y[None, None, :])
    if wp % 2 == 0:
        pxe[:, :, wp // 2] = np.cos(L2("3.14159265358979323846264338327950") * pu.astype(L2)).astype(np.float64)
    if hp % 2 == 0:
        pye[:, :, hp // 2] = np.cos(L2("3.14159265358979323846264338327950") * pv.astype(L2)).astype(np.float64)
    Ae = fdl.construct._system_chunk(pu, pv, pxe, pye, vs, d, grid, kx, ky)
    reg = (grid.omega_x[kx] ** 2 + grid.omega_y[ky] ** 2)[:, None] ** 2 * d[None, :] ** 4 + 1e-9

    def normal(AA):
        AH = AA.conj().transpose(0, 2, 1)
        G = AH @ AA
        G[:, np.arange(n), np.arange(n)] += lam * reg
        return G, AH @ b_all[q]

    G, rhs = normal(A)
    x = np.linalg.solve(G, rhs)
    Lc = np.linalg.cholesky(G)
    x_ch = np.stack([sla.cho_solve((Lc[i], True), rhs[i]) for i in range(len(q))])
    rev = np.arange(n)[::-1]
    x_rev = np.linalg.solve(G[:, rev][:, :, rev], rhs[:, rev])[:, np.argsort(rev)]
    Ge, rhse = normal(Ae)
    x_ph = np.linalg.solve(Ge, rhse)
    f = lambda y: float(np.linalg.norm(y - x) / np.linalg.norm(x))
    return np.array([f(x_ch), f(x_rev), f(x_ph)])


def construct_case(name, views32, u, v, d, render_uv, lam=None, pad=None, s=None, ap=None, **extra):
    m = views32.shape[0]
    aps = [ap] * m if ap is not None else None
    vs = ViewSet(images=views32.astype(np.float64), u=u, v=v, s=s, apertures=aps)
    sh = ShiftParams.factored(u, v, d)
    kw = {} if pad is None else {"pad_margin": pad}
    model = construct_fdl(vs, sh, lam=lam, **kw)
    renders = np.stack([render(model, RenderRequest(u=a, v=b, f=0.0)) for a, b in render_uv])
    fl = floors(views32, np.outer(u, d), np.outer(v, d), np.asarray(d, float), model.lambda_used,
                model.pad_margin, aps=aps, s=s)
    print(name, "floors (chol, rev, phase):", fl)
    save(name, floor=fl, views=views32, u=u, v=v, d=d, s=(s if s is not None else np.zeros(m)),
         lam_in=np.array(np.nan if lam is None else lam), pad_in=np.array(-1 if pad is None else pad),
         layers=model.layers, lam=np.array(model.lambda_used), pad=np.array(model.pad_margin),
         render_uv=np.asarray(render_uv, dtype=np.float64), renders=renders, **ap_fields("ap", ap), **extra)


def main():
    # C1 at full size (config 1)
    c1 = make_case("c1")
    sel = np.array([0, 6, 12, 18, 24])
    construct_case("c1_full", c1.views.numpy(), c1.u, c1.v, c1.d, c1.render_coords[sel])

    # C2 layout (9x9 RGB, n=30, d in [-3, 3]) at 24 px
    c2 = make_case("c2", 24)
    uv = np.array([[0.0, 0.0], [4.0, -3.0], [0.5, 0.5], [-3.5, 2.5]])
    construct_case("c2_s24", c2.views.numpy(), c2.u, c2.v, c2.d, uv)

    # C3 layout: focal stack of 40 disk(8) images at 32 px, n = 48 (real-A path)
    rng = np.random.default_rng(3)
    h = w = 32
    d3 = np.linspace(-4, 4, 48)
    ap8 = aperture_spectrum("disk", diameter=8.0)
    gt = np.fft.rfft2(rng.uniform(0, 1, (48, 1, h, w)) / 48.0, axes=(-2, -1))
    gt_model = FdlModel(disparities=d3, layers=gt, grid=FrequencyGrid(w, h), width=w, height=h)
    focus = np.linspace(-4, 4, 40)
    focal = np.stack([render(gt_model, RenderRequest(u=0.0, v=0.0, s=fi, f=1.0, aperture=ap8))
                      for fi in focus]).astype(np.float32)
    construct_case("c3_s32", focal, np.zeros(40), np.zeros(40), d3, grid_coords(3, spacing=4.0)[[0, 4, 8]],
                   s=focus, ap=ap8)

    # C4 layout (17x17 RGB views, n = 64, d in [-6, 6]) at 16 px: sampled bins only
    c4 = make_case("c4", 16)
    views = c4.views.numpy()
    vs = ViewSet(images=views.astype(np.float64), u=c4.u, v=c4.v)
    pu, pv = np.outer(c4.u, c4.d), np.outer(c4.v, c4.d)
    pad = int(np.ceil(max(np.abs(pu).max(), np.abs(pv).max())))
    img = np.pad(vs.images, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    hp, wp = img.shape[1:3]
    whp = wp // 2 + 1
    spec = np.fft.rfft2(np.moveaxis(img, 3, 1), axes=(-2, -1))
    b_all = spec.reshape(len(c4.u), 3, hp * whp).transpose(2, 0, 1)
    lam = fdl.construct.default_lambda(np.sum(np.abs(b_all) ** 2, axis=(1, 2)), len(c4.u))
    grid = FrequencyGrid(wp, hp)
    px, py = fdl.construct._phase_tables(pu, pv, grid)
    srng = np.random.default_rng(44)
    q = np.sort(srng.choice(hp * whp, 192, replace=False))
    kx, ky = q % whp, q // whp
    A = fdl.construct._system_chunk(pu, pv, px, py, vs, c4.d, grid, kx, ky)
    reg = (grid.omega_x[kx] ** 2 + grid.omega_y[ky] ** 2)[:, None] ** 2 * c4.d[None, :] ** 4 + 1e-9
    x = fdl.construct._solve_chunk(A, b_all[q], reg, lam, grid, kx, ky)
    fl = floors(views, pu, pv, c4.d, lam, pad, bins=q)
    print("c4 floors", fl)
    save("c4_s16_bins", floor=fl, views=views, u=c4.u, v=c4.v, d=c4.d, lam=np.array(lam), pad=np.array(pad),
         bins=q, x=x)

    # render-only: C5-like random FDL with disk(1) requests f = 2r, plus pinhole
    n5, h5, w5 = 16, 30, 40
    lay = random_fdl_layers(n5, 3, h5, w5, seed=55, dtype=__import__("torch").complex128).numpy()
    d5 = np.linspace(-5, 5, n5)
    model5 = FdlModel(disparities=d5, layers=lay, grid=FrequencyGrid(w5, h5), width=w5, height=h5)
    ap1 = aperture_spectrum("disk", diameter=1.0)
    u, v, s, f = render_requests_c5(10, seed=55)
    f[0] = 0.0  # one pinhole request
    f[1] = 40.0  # a wide one that runs off the table (OOB lookups)
    outs, ops, oob = [], [], []
    for i in range(len(u)):
        ap1.oob_count = 0
        outs.append(render(model5, RenderRequest(u=u[i], v=v[i], s=s[i], f=f[i], aperture=ap1)))
        st = last_render_stats()
        ops.append(st.layer_ops)
        oob.append(st.oob_lookups)
    save("render_c5_small", layers=lay, d=d5, u=u, v=v, s=s, f=f, renders=np.stack(outs),
         layer_ops=np.array(ops), oob=np.array(oob), **ap_fields("ap", ap1))

    # polygon (complex table) + square apertures, odd grid, uncropped, gamma
    n6, h6, w6 = 5, 17, 15
    lay6 = np.fft.rfft2(np.random.default_rng(6).uniform(0, 0.2, (n6, 2, h6, w6)), axes=(-2, -1))
    d6 = np.array([-2.0, -0.5, 0.0, 1.0, 2.5])
    m6 = FdlModel(disparities=d6, layers=lay6, grid=FrequencyGrid(w6, h6), width=w6 - 2, height=h6 - 2,
                  pad_margin=1, color_space="linear")
    verts = [(np.cos(a), np.sin(a)) for a in np.linspace(0, 2 * np.pi, 6)[:-1]]
    poly = aperture_spectrum("polygon", vertices=verts, pad_factor=4)
    sq = aperture_spectrum("square", side=0.5, pad_factor=4)
    reqs = [dict(u=0.3, v=-1.2, s=0.4, f=2.0, ap="poly", gamma="as-stored", crop=True),
            dict(u=-0.7, v=0.2, s=-1.0, f=1.5, ap="sq", gamma="linear-process", crop=True),
            dict(u=1.1, v=0.9, s=0.0, f=0.0, ap="poly", gamma="as-stored", crop=False)]
    outs6 = []
    for r in reqs:
        ap = poly if r["ap"] == "poly" else sq
        outs6.append(render(m6, RenderRequest(u=r["u"], v=r["v"], s=r["s"], f=r["f"], aperture=ap,
                                              gamma_mode=r["gamma"], crop=r["crop"])))
    save("render_apertures", layers=lay6, d=d6, pad=np.array(1), req_u=np.array([r["u"] for r in reqs]),
         req_v=np.array([r["v"] for r in reqs]), req_s=np.array([r["s"] for r in reqs]),
         req_f=np.array([r["f"] for r in reqs]), render0=outs6[0], render1=outs6[1], render2=outs6[2],
         **ap_fields("poly", poly), **ap_fields("sq", sq))

    # reference test scene (tests/conftest.py:39-52): asymmetric d -> the complex path
    trng = np.random.default_rng(1234)
    scene = SceneSpec(masks=quadrant_masks(64, 64, 4), disparities=[-1.0, 0.0, 1.0, 2.0],
                      texture=smooth_texture(trng, 64, 64))
    lv = synthesize_lightfield(scene, grid_coords(3))
    views_l = lv.images.astype(np.float32)
    construct_case("lambertian_lam1e-6", views_l, lv.u, lv.v, np.array([-1.0, 0.0, 1.0, 2.0]),
                   np.array([[0.0, 0.0], [1.0, -1.0], [2.0, 1.0]]), lam=1e-6, pad=0)
    construct_case("lambertian_default", views_l, lv.u, lv.v, np.array([-1.0, 0.0, 1.0, 2.0]),
                   np.array([[0.0, 0.0], [0.5, -0.5]]))

    # odd sizes, odd symmetric n (middle layer), relaxed shifts + render_views_with_shifts
    c1o = make_case("c1", (21, 19), side=3)
    d_odd = np.linspace(-1.0, 1.0, 5)
    construct_case("odd_grid_n5", c1o.views.numpy(), c1o.u, c1o.v, d_odd, np.array([[0.0, 0.0], [1.0, 1.0]]))
    prng = np.random.default_rng(7)
    pu = np.outer(c1o.u, d_odd) + 0.05 * prng.standard_normal((9, 5))
    pv = np.outer(c1o.v, d_odd) + 0.05 * prng.standard_normal((9, 5))
    vs = ViewSet(images=c1o.views.numpy().astype(np.float64), u=c1o.u, v=c1o.v)
    rel = ShiftParams.relaxed(pu, pv, d=d_odd)
    mrel = construct_fdl(vs, rel, lam=1e-3)
    stack = render_views_with_shifts(mrel, rel)
    fl = floors(c1o.views.numpy(), pu, pv, d_odd, mrel.lambda_used, mrel.pad_margin)
    print("relaxed floors", fl)
    save("relaxed_n5", floor=fl, views=c1o.views.numpy(), u=c1o.u, v=c1o.v, d=d_odd, pu=pu, pv=pv,
         layers=mrel.layers, lam=np.array(mrel.lambda_used), pad=np.array(mrel.pad_margin), stack=stack)


if __name__ == "__main__":
    main()

"""The reference package's own construct/render tests, run against the B200 path.

Ports of the reference's tests/test_construct.py (class TestConstruct),
tests/test_render.py (TestRender, TestRenderWithShifts) and the acceptance
criteria 1, 4, 6 and 8 (tests/test_acceptance.py), with the reference's
fixtures (tests/conftest.py: smooth_texture, quadrant_masks, grid_coords and
the 4-layer 64x64 Lambertian scene) restated here and its synthetic light-field
generator restated in oracle/fdl_oracle.py (layered_views).

Tolerances: where the reference asserts 1e-10 / 1e-12 / 1e-8 agreement it
relies on float64 renders of complex128 layers; this implementation stores
complex64 layers and renders in float32 (BASELINE.json north_star: fp32
tolerances), so those asserts are relaxed to 1e-5-level and say so; every
array_equal / bitwise contract (f = 0 ignores aperture and s, pinhole ignores
s, chunk independence) is kept exactly.
"""

import time

import numpy as np
import pytest

from conftest import psnr
from oracle import fdl_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fdl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_06919_b200 as pkg
    return pkg


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


def grid_coords(side=3, spacing=1.0):
    g = (np.arange(side) - (side - 1) / 2) * spacing
    return np.array([(u, v) for v in g for u in g])


def lambertian(fdl, rng, coords=None, h=64, k=4, disp=(-1.0, 0.0, 1.0, 2.0)):
    coords = grid_coords(3) if coords is None else coords
    masks = quadrant_masks(h, h, k)
    tex = smooth_texture(rng, h, h)
    imgs = O.layered_views(masks, disp[:k], tex, coords)
    return fdl.ViewSet(images=imgs, u=coords[:, 0], v=coords[:, 1]), np.array(disp[:k]), masks, tex


def model_of(fdl, views, d, lam=1e-6, pad=0):
    return fdl.construct_fdl(views, fdl.ShiftParams.factored(views.u, views.v, d), lam=lam, pad_margin=pad)


# ------------------------------------------------------------------ TestConstruct
def test_single_view_single_layer_identity(fdl):
    rng = np.random.default_rng(1234)
    img = rng.uniform(0, 1, (1, 16, 16, 1))
    model = fdl.construct_fdl(fdl.ViewSet(images=img, u=[0.0], v=[0.0]),
                              fdl.ShiftParams.factored([0.0], [0.0], [0.0]), lam=0.0, pad_margin=0)
    expected = np.fft.rfft2(img[0, :, :, 0])
    # reference: < 1e-9 absolute in complex128; complex64 layers -> relative 1e-6
    assert np.max(np.abs(model.layers[0, 0] - expected)) < 1e-6 * np.max(np.abs(expected))


def test_constant_image_two_views(fdl):
    img = np.full((2, 8, 8, 1), 0.5)
    views = fdl.ViewSet(images=img, u=[0.0, 1.0], v=[0.0, 0.0])
    model = fdl.construct_fdl(views, fdl.ShiftParams.factored(views.u, views.v, [0.0, 1.0]), lam=1e-3, pad_margin=0)
    for u in (0.0, 1.0):
        out = fdl.render(model, fdl.RenderRequest(u=u, v=0.0, f=0.0))
        assert np.max(np.abs(out - 0.5)) < 1e-6


def test_round_trip_exact_recovery(fdl):
    views, d, _, _ = lambertian(fdl, np.random.default_rng(1234))
    model = model_of(fdl, views, d)
    for j, (u, v) in enumerate(zip(views.u, views.v)):
        out = fdl.render(model, fdl.RenderRequest(u=u, v=v, f=0.0))
        assert psnr(out, views.images[j][:, :, 0]) >= 80.0


def test_overparameterized_rejected_without_regularization(fdl):
    views, _, _, _ = lambertian(fdl, np.random.default_rng(1234))
    with pytest.raises(fdl.RankDeficiencyError):
        fdl.construct_fdl(views, fdl.ShiftParams.factored(views.u, views.v, np.linspace(-2, 2, 12)), lam=0.0)


def test_chunk_independence_bitwise(fdl):
    rng = np.random.default_rng(1234)
    views, d, _, _ = lambertian(fdl, rng, h=16, k=2, disp=(0.0, 1.0))
    sh = fdl.ShiftParams.factored(views.u, views.v, d)
    models = [fdl.construct_fdl(views, sh, lam=1e-4, pad_margin=0, chunk=c) for c in (7, 64, 10 ** 6)]
    for m2 in models[1:]:
        assert np.array_equal(models[0].layers, m2.layers)


def test_monotone_fit_in_lambda(fdl):
    rng = np.random.default_rng(1234)
    views, _, _, _ = lambertian(fdl, rng, h=16, k=2, disp=(0.0, 1.0))
    sh = fdl.ShiftParams.factored(views.u, views.v, [-0.5, 0.5, 1.5])
    energy = float(np.sum(views.images ** 2))

    def residual(lam):
        model = fdl.construct_fdl(views, sh, lam=lam, pad_margin=0)
        return sum(float(np.sum((fdl.render(model, fdl.RenderRequest(u=u, v=v)) - views.images[j][:, :, 0]) ** 2))
                   for j, (u, v) in enumerate(zip(views.u, views.v)))

    res = [residual(lam) for lam in (10.0, 1.0, 1e-2, 1e-4, 1e-6)]
    for a, b in zip(res, res[1:]):
        # reference: b <= a (1 + 1e-9) in float64.  An fp32 render error d
        # (|d| <= 1e-6 |image| in rms) moves sum r^2 by at most
        # 2 |r| |d| (Cauchy-Schwarz), hence the extra term.
        assert b <= a * (1 + 1e-9) + 2e-6 * np.sqrt(a * energy)


def test_ridge_limit_decay(fdl):
    rng = np.random.default_rng(1234)
    views, _, _, _ = lambertian(fdl, rng, h=16, k=2, disp=(0.0, 1.0))
    d = np.array([-0.5, 0.5, 1.5])
    sh = fdl.ShiftParams.factored(views.u, views.v, d)
    models = [fdl.construct_fdl(views, sh, lam=lam, pad_margin=0) for lam in (1e-6, 1e-2, 1e2, 1e6)]
    g = models[0].grid
    osq = (g.omega_x[None, :] ** 2 + g.omega_y[:, None] ** 2) ** 2
    weight = osq[None] * (d ** 4)[:, None, None]
    strong = weight >= 1e-4
    energies = [float(np.sum(np.abs(m.layers[:, 0][strong]) ** 2)) for m in models]
    for a, b in zip(energies, energies[1:]):
        assert b <= a * (1 + 1e-6)
    assert energies[-1] < 1e-3 * energies[0]


def test_pinhole_ignores_refocus_parameter(fdl):
    views_a, d, _, _ = lambertian(fdl, np.random.default_rng(1234))
    views_b = fdl.ViewSet(images=views_a.images.copy(), u=views_a.u, v=views_a.v, s=np.full(9, 7.3))
    sh = fdl.ShiftParams.factored(views_a.u, views_a.v, d)
    m_a = fdl.construct_fdl(views_a, sh, lam=1e-4, pad_margin=0)
    m_b = fdl.construct_fdl(views_b, sh, lam=1e-4, pad_margin=0)
    assert np.array_equal(m_a.layers, m_b.layers)


def test_focal_stack_input_path(fdl):
    rng = np.random.default_rng(1234)
    masks = quadrant_masks(32, 32, 2)
    tex = smooth_texture(rng, 32, 32)
    dense_coords = grid_coords(5, spacing=0.5)
    dense = O.layered_views(masks, [0.0, 1.0], tex, dense_coords)
    focal = np.stack([np.atleast_3d(O.refocus_shift_and_sum(dense, dense_coords[:, 0], dense_coords[:, 1], s))
                      for s in (0.0, 1.0)])
    ap = fdl.aperture_spectrum("square", side=2.0, pad_factor=8, resolution=128)
    stack = fdl.ViewSet(images=focal, u=[0.0, 0.0], v=[0.0, 0.0], s=[0.0, 1.0], apertures=[ap, ap])
    model = fdl.construct_fdl(stack, fdl.ShiftParams.factored([0.0, 0.0], [0.0, 0.0], [0.0, 1.0]),
                              lam=1e-4, pad_margin=0)
    assert fdl.last_construct_stats().path == 2
    for j, s in enumerate((0.0, 1.0)):
        out = fdl.render(model, fdl.RenderRequest(u=0.0, v=0.0, s=s, f=1.0, aperture=ap))
        assert psnr(out, focal[j][:, :, 0]) > 30.0


def test_relaxed_shifts_need_disparities(fdl):
    views, _, _, _ = lambertian(fdl, np.random.default_rng(1234))
    with pytest.raises(ValueError, match="disparities"):
        fdl.construct_fdl(views, fdl.ShiftParams.relaxed(np.zeros((9, 2)), np.zeros((9, 2))), lam=1e-4)


def test_pad_margin_recorded_and_cropped(fdl):
    views, d, _, _ = lambertian(fdl, np.random.default_rng(1234))
    model = fdl.construct_fdl(views, fdl.ShiftParams.factored(views.u, views.v, d), lam=1e-4)
    assert model.pad_margin == 2 and model.grid.width == views.width + 4
    assert fdl.render(model, fdl.RenderRequest()).shape == (views.height, views.width)


# ------------------------------------------------------------------ TestRender
def test_single_zero_disparity_layer_is_identity(fdl):
    rng = np.random.default_rng(1234)
    img = rng.uniform(0, 1, (16, 16))
    spec = np.fft.rfft2(img)[None, None]
    model = fdl.FdlModel(disparities=np.array([0.0]), layers=spec, grid=fdl.FrequencyGrid(16, 16), width=16, height=16)
    ap = fdl.aperture_spectrum("disk", diameter=1.0, pad_factor=8)
    for (u, v, s, f) in [(0.0, 0.0, 0.0, 0.0), (1.5, -2.0, 0.0, 0.0), (0.3, 0.4, 0.0, 1.0), (0.0, 0.0, 0.0, 2.0)]:
        out = fdl.render(model, fdl.RenderRequest(u=u, v=v, s=s, f=f, aperture=ap))
        assert np.max(np.abs(out - img)) < 1e-5  # reference: 1e-10 in float64


def test_matches_spatial_shift_oracle_integer(fdl):
    views, d, _, _ = lambertian(fdl, np.random.default_rng(1234))
    model = model_of(fdl, views, d)
    lay = [O.half_inverse(model.layers[k], 64, 64) for k in range(len(d))]
    for (u0, v0) in [(2.0, 1.0), (-1.0, 2.0), (0.0, -3.0), (1.0, 1.0)]:
        out = fdl.render(model, fdl.RenderRequest(u=u0, v=v0, f=0.0))
        oracle = sum(np.roll(lay[k], (int(-v0 * dk), int(-u0 * dk)), axis=(0, 1)) for k, dk in enumerate(d))
        assert np.sqrt(np.mean((out - oracle) ** 2)) <= 1e-5  # reference: 1e-8 in float64


def test_linearity_in_model(fdl):
    rng = np.random.default_rng(1234)
    g = fdl.FrequencyGrid(16, 16)
    la = np.fft.rfft2(rng.uniform(0, 1, (2, 1, 16, 16)), axes=(-2, -1))
    lb = np.fft.rfft2(rng.uniform(0, 1, (2, 1, 16, 16)), axes=(-2, -1))
    d = np.array([-0.5, 1.0])
    req = fdl.RenderRequest(u=0.7, v=-0.3, s=0.2, f=1.0, aperture=fdl.aperture_spectrum("disk", diameter=1.0))
    mk = lambda L: fdl.FdlModel(disparities=d, layers=L, grid=g, width=16, height=16)
    out = fdl.render(mk(la + lb), req)
    assert np.allclose(out, fdl.render(mk(la), req) + fdl.render(mk(lb), req), atol=1e-5)


def test_f_zero_ignores_aperture_and_s(fdl):
    views, d, _, _ = lambertian(fdl, np.random.default_rng(1234))
    model = model_of(fdl, views, d)
    outs = [fdl.render(model, fdl.RenderRequest(u=0.5, v=0.5, s=s, f=0.0, aperture=ap))
            for s, ap in [(0.0, None), (3.0, fdl.aperture_spectrum("disk", diameter=2.0)),
                          (-1.0, fdl.aperture_spectrum("square", side=0.5))]]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_aperture_scale_continuity_at_zero(fdl):
    views, d, _, _ = lambertian(fdl, np.random.default_rng(1234))
    model = model_of(fdl, views, d)
    ap = fdl.aperture_spectrum("disk", diameter=1.0, pad_factor=8)
    r0 = fdl.render(model, fdl.RenderRequest(u=0.3, v=-0.2, s=0.5, f=0.0, aperture=ap))
    r1 = fdl.render(model, fdl.RenderRequest(u=0.3, v=-0.2, s=0.5, f=1e-4, aperture=ap))
    assert np.max(np.abs(r0 - r1)) < 1e-3


def test_render_matches_grid_sampled_shift_and_sum(fdl):
    views, d, _, _ = lambertian(fdl, np.random.default_rng(1234))
    model = model_of(fdl, views, d)
    n = 15
    raster = np.zeros((n, n))
    idx = (np.array([-1.0, 0.0, 1.0]) / 0.2 + (n - 1) / 2).astype(int)
    for iy in idx:
        for ix in idx:
            raster[iy, ix] = 1.0
    ap = fdl.aperture_spectrum("raster", image=raster, extent=3.0, pad_factor=64)
    ceiling = min(psnr(fdl.render(model, fdl.RenderRequest(u=u, v=v)), views.images[j][:, :, 0])
                  for j, (u, v) in enumerate(zip(views.u, views.v)))
    for s in (0.0, 1.0, -1.0):
        got = fdl.render(model, fdl.RenderRequest(u=0.0, v=0.0, s=s, f=1.0, aperture=ap))
        oracle = O.refocus_shift_and_sum(views.images, views.u, views.v, s)
        # reference: >= ceiling - 1 dB with a float64 ceiling (~150+ dB); fp32 renders saturate ~120 dB
        assert psnr(got, oracle) >= min(ceiling, 100.0) - 1.0


def test_cost_independent_of_view_count(fdl):
    rng = np.random.default_rng(1234)
    v9, d, _, _ = lambertian(fdl, rng)
    v25, _, _, _ = lambertian(fdl, np.random.default_rng(1234), coords=grid_coords(5, spacing=0.5))
    req = fdl.RenderRequest(u=0.2, v=0.1, s=0.5, f=1.0, aperture=fdl.aperture_spectrum("disk", diameter=1.0))
    fdl.render(model_of(fdl, v9, d), req)
    ops9 = fdl.last_render_stats().layer_ops
    fdl.render(model_of(fdl, v25, d), req)
    assert ops9 == fdl.last_render_stats().layer_ops


def test_gamma_mode(fdl):
    views, d, _, _ = lambertian(fdl, np.random.default_rng(1234))
    with pytest.raises(ValueError, match="linear"):
        fdl.render(model_of(fdl, views, d), fdl.RenderRequest(gamma_mode="linear-process"))
    rng = np.random.default_rng(1234)
    img = rng.uniform(0.05, 0.95, (8, 8))
    lin = fdl.srgb_decode(img)
    views = fdl.ViewSet(images=lin[None, :, :, None], u=[0.0], v=[0.0], color_space=fdl.LINEAR)
    model = fdl.construct_fdl(views, fdl.ShiftParams.factored([0.0], [0.0], [0.0]), lam=0.0, pad_margin=0)
    out = fdl.render(model, fdl.RenderRequest(gamma_mode="linear-process"))
    assert np.max(np.abs(out - img)) < 1e-5  # reference: 1e-8 in float64


def test_render_views_with_shifts_matches_render(fdl):
    views, d, _, _ = lambertian(fdl, np.random.default_rng(1234))
    model = model_of(fdl, views, d)
    stack = fdl.render_views_with_shifts(model, fdl.ShiftParams.factored(views.u, views.v, d))
    for j, (u, v) in enumerate(zip(views.u, views.v)):
        assert np.max(np.abs(stack[j] - fdl.render(model, fdl.RenderRequest(u=u, v=v)))) < 1e-12


# ------------------------------------------------------------------ acceptance criteria
def test_criterion_1_exact_recovery_round_trip(fdl):
    rng = np.random.default_rng(10)
    t0 = time.perf_counter()
    views, d, _, _ = lambertian(fdl, rng)
    model = model_of(fdl, views, d)
    worst = min(psnr(fdl.render(model, fdl.RenderRequest(u=u, v=v)), views.images[j][:, :, 0])
                for j, (u, v) in enumerate(zip(views.u, views.v)))
    assert worst >= 80.0 and time.perf_counter() - t0 < 5.0


def test_criterion_6_layer_count_saturation(fdl):
    rng = np.random.default_rng(60)
    masks = quadrant_masks(48, 48, 4)
    tex = smooth_texture(rng, 48, 48)
    gg = np.linspace(-1, 1, 11)
    coords = np.array([(u, v) for v in gg for u in gg])
    clean = O.layered_views(masks, [-1.0, 0.0, 1.0, 2.0], tex, coords)
    noisy = fdl.ViewSet(images=clean + 0.01 * rng.standard_normal(clean.shape), u=coords[:, 0], v=coords[:, 1])
    priority = [0.0, -1.0, 1.0, 2.0, 0.5, -0.5, 1.5, -1.5]

    def round_trip(n):
        d = np.sort(priority[:n])
        m = fdl.construct_fdl(noisy, fdl.ShiftParams.factored(noisy.u, noisy.v, d), lam=None, pad_margin=0)
        imgs = fdl.render_many(m, [fdl.RenderRequest(u=u, v=v) for u, v in coords])
        return float(np.mean([psnr(imgs[j], noisy.images[j][:, :, 0]) for j in range(len(coords))]))

    curve = [round_trip(n) for n in range(1, 9)]
    assert all(b >= a - 0.01 for a, b in zip(curve[:4], curve[1:4]))
    assert max(abs(p - curve[3]) for p in curve[4:]) < 0.2


def test_criterion_8_performance_budgets(fdl):
    rng = np.random.default_rng(80)
    views = fdl.ViewSet(images=rng.uniform(0, 1, (9, 512, 512, 1)), u=np.tile([-1.0, 0.0, 1.0], 3),
                        v=np.repeat([-1.0, 0.0, 1.0], 3))
    sh = fdl.ShiftParams.factored(views.u, views.v, np.linspace(-2, 2, 20))
    fdl.construct_fdl(views, sh, lam=1e-4, pad_margin=0)  # warm-up (plans, allocator)
    t0 = time.perf_counter()
    model = fdl.construct_fdl(views, sh, lam=1e-4, pad_margin=0)
    construct_s = time.perf_counter() - t0
    req = fdl.RenderRequest(u=0.3, v=-0.2, s=0.5, f=1.0, aperture=fdl.aperture_spectrum("disk", diameter=1.0))
    fdl.render(model, req)
    render_ms = min((lambda t: (fdl.render(model, req), (time.perf_counter() - t) * 1e3)[1])(time.perf_counter())
                    for _ in range(3))
    print(f"criterion 8: construction {construct_s * 1e3:.1f} ms (budget 30 s), render {render_ms:.2f} ms (budget 100 ms)")
    assert construct_s <= 30.0 and render_ms <= 100.0

"""K0 / K4 through the library's FFT engine (csrc/fft2.cuh, k0_fft.cu)
against numpy's pocketfft (what the reference calls: construct.py:261-263,
spectra.py:202-208) and against the cuFFT path of the same entry points.

The engine serves grids whose sides are 67 * 2^a or 131 * 2^a (C1 134, C2
536, C2b 1048, C4 2144); fdl_fft_force_cufft(1) (a test hook of the C ABI)
forces the cuFFT path on this thread.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import importlib
    K = importlib.import_module("paper_1901_06919_b200.construct")
    R = importlib.import_module("paper_1901_06919_b200.render")
    return torch, K, R


def _with_fft(mode, fn):
    """mode "engine": the library's default (its engine where it applies); "cufft": forced cuFFT."""
    from paper_1901_06919_b200 import _native
    lib = _native.lib()
    lib.fdl_fft_force_cufft(1 if mode == "cufft" else 0)
    try:
        return fn()
    finally:
        lib.fdl_fft_force_cufft(0)


# (m, H, W, C, pad): padded sides 134, 536, 1048, 2144 and non-square 134 x 268, 524 x 134
FWD_CASES = [
    (3, 128, 128, 1, 3),
    (4, 512, 512, 3, 12),
    (2, 128, 262, 3, 3),
    (2, 518, 128, 2, 3),
    (3, 110, 110, 4, 12),
    (2, 1024, 1024, 1, 12),
    (1, 2048, 2048, 3, 48),
]


@pytest.mark.parametrize("m,H,W,C,pad", FWD_CASES)
def test_engine_forward_matches_numpy(env, m, H, W, C, pad):
    torch, K, _ = env
    rng = np.random.default_rng(H * 7 + W)
    views = rng.uniform(0, 1, (m, H, W, C)).astype(np.float32)
    spec, sumsq = _with_fft("engine", lambda: K.views_to_spectra(torch.from_numpy(views).cuda(), pad))
    got = spec.cpu().numpy()
    padded = np.pad(views.astype(np.float64), ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    ref = np.moveaxis(np.fft.rfft2(padded, axes=(1, 2)), 3, 1)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    cuf = _with_fft("cufft", lambda: K.views_to_spectra(torch.from_numpy(views).cuda(), pad))[0].cpu().numpy()
    err_cufft = np.linalg.norm(cuf - ref) / np.linalg.norm(ref)
    print(f"fwd {m}x{H}x{W}x{C} pad {pad}: engine rel err {err:.3e}, cufft {err_cufft:.3e}")
    # fp32 transforms: within 2x of cuFFT's own error against fp64 numpy
    assert err < max(2e-7, 2 * err_cufft), (err, err_cufft)
    assert np.max(np.abs(got - ref)) < 2e-6 * np.max(np.abs(ref))
    ref_ss = np.sum(np.abs(ref) ** 2, axis=(1, 2, 3))
    np.testing.assert_allclose(sumsq.cpu().numpy(), ref_ss, rtol=1e-6)


@pytest.mark.parametrize("m,H,W,C,pad", FWD_CASES[:3])
def test_engine_forward_agrees_with_cufft(env, m, H, W, C, pad):
    torch, K, _ = env
    rng = np.random.default_rng(5)
    views = torch.from_numpy(rng.uniform(0, 1, (m, H, W, C)).astype(np.float32)).cuda()
    a, sa = _with_fft("engine", lambda: K.views_to_spectra(views, pad))
    b, sb = _with_fft("cufft", lambda: K.views_to_spectra(views, pad))
    err = (torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b)).item()
    assert err < 4e-7, err  # two independent fp32 errors of ~1.6e-7 each
    np.testing.assert_allclose(sa.cpu().numpy(), sb.cpu().numpy(), rtol=1e-6)


def test_engine_forward_batch_independent(env):
    """Every view's spectrum is bit-identical however the views are batched
    (the multi-GPU view sharding and the chunked upload rely on it)."""
    torch, K, _ = env
    rng = np.random.default_rng(9)
    views = torch.from_numpy(rng.uniform(0, 1, (5, 512, 512, 3)).astype(np.float32)).cuda()
    full, s_full = _with_fft(None, lambda: K.views_to_spectra(views, 12))
    for j0, j1 in [(0, 1), (1, 4), (4, 5)]:
        part, s_part = _with_fft(None, lambda: K.views_to_spectra(views[j0:j1].contiguous(), 12))
        assert torch.equal(part, full[j0:j1])
        assert torch.equal(s_part, s_full[j0:j1])


INV_CASES = [
    (3, 1, 134, 134, 3, False),
    (4, 3, 536, 536, 12, False),
    (2, 3, 536, 536, 12, True),
    (2, 3, 134, 268, 27, False),
    (2, 2, 524, 134, 3, False),
    (2, 4, 268, 134, 0, False),
    (1, 1, 1048, 1048, 12, False),
    (1, 3, 2144, 2144, 48, False),
    # mixed-radix engine (csrc/fft_mr.cuh, k4_mr.cu): config 5's 1920 x 1080 grid, both orientations,
    # odd view / channel counts (ragged tiles), a crop and the sRGB epilogue
    (2, 3, 1080, 1920, 0, False),
    (1, 1, 1080, 1920, 0, True),
    (3, 2, 1920, 1080, 4, False),
    (1, 4, 1080, 1080, 7, False),
]


@pytest.mark.parametrize("V,C,Hp,Wp,pad,srgb", INV_CASES)
def test_engine_inverse_matches_numpy(env, V, C, Hp, Wp, pad, srgb):
    torch, _, R = env
    rng = np.random.default_rng(Hp + Wp + C)
    # spectra of real images plus a non-Hermitian perturbation on the
    # self-conjugate columns (numpy's irfft2 drops its imaginary part there)
    img = rng.uniform(0, 1, (V, C, Hp, Wp))
    spec = np.fft.rfft2(img, axes=(2, 3))
    spec[..., 0] += 1e-2 * (rng.standard_normal((V, C, Hp)) * 1j) * np.abs(spec[..., 0]).mean()
    Ho, Wo = Hp - 2 * pad, Wp - 2 * pad
    dev = torch.from_numpy(spec.astype(np.complex64)).cuda()
    got = _with_fft("engine", lambda: R.spectra_to_images(dev.clone(), Hp, Wp, pad, Ho, Wo, srgb=srgb)).cpu().numpy()
    ref = np.fft.irfft2(spec.astype(np.complex64).astype(np.complex128), s=(Hp, Wp), axes=(2, 3))
    ref = np.moveaxis(ref[:, :, pad:pad + Ho, pad:pad + Wo], 1, 3)
    if srgb:
        x = np.maximum(ref, 0)
        ref = np.where(x <= 0.0031308, 12.92 * x, 1.055 * x ** (1 / 2.4) - 0.055)
    cuf = _with_fft("cufft", lambda: R.spectra_to_images(dev.clone(), Hp, Wp, pad, Ho, Wo, srgb=srgb)).cpu().numpy()
    e_eng, e_cuf = np.max(np.abs(got - ref)), np.max(np.abs(cuf - ref))
    print(f"inv {V}x{C}x{Hp}x{Wp} pad {pad} srgb {srgb}: engine max err {e_eng:.3e}, cufft {e_cuf:.3e}")
    assert e_eng < max(2e-6, 2 * e_cuf), (e_eng, e_cuf)

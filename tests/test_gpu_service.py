"""GPU-resident pipeline pieces and the render-service backend (SURVEY.md §8(f)
row 2): K6 against numpy, one upload per pipeline run, device-side
quantisation, and the reference's service contract (serve.py:86-143; cases of
the reference's tests/test_serve.py that do not need the HTTP front end)."""

import io
import json
import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def g():
    return load_golden("pipeline")


def _views(g, dtype=np.float64):
    from paper_1901_06919_b200 import ViewSet
    return ViewSet(images=g["images"].astype(dtype), u=g["coords"][:, 0], v=g["coords"][:, 1])


def _known(g):
    from paper_1901_06919_b200 import ShiftParams
    return ShiftParams.factored(g["coords"][:, 0], g["coords"][:, 1], g["d"])


@pytest.mark.parametrize("C", [1, 3])
@pytest.mark.parametrize("ref_dtype", [np.float32, np.float64])
def test_view_sqerr_matches_numpy(torch_cuda, C, ref_dtype):
    torch = torch_cuda
    from paper_1901_06919_b200 import ViewSet
    from paper_1901_06919_b200.pipeline import ResidentViews
    rng = np.random.default_rng(3)
    ref = rng.uniform(0, 1, (5, 37, 41, C)).astype(ref_dtype)
    out = (ref + rng.normal(0, 0.01, ref.shape)).astype(np.float32)
    res = ResidentViews(ViewSet(images=ref, u=np.zeros(5), v=np.zeros(5)))
    sq = res.squared_errors(torch.as_tensor(out, device="cuda"))
    want = ((out.astype(np.float64) - ref.astype(np.float64)) ** 2).sum(axis=(1, 2))
    np.testing.assert_allclose(sq, want, rtol=1e-12)
    assert res.uploaded_bytes == ref.nbytes


def test_quantise_u8_is_numpy_round(torch_cuda):
    torch = torch_cuda
    from paper_1901_06919_b200.serve import quantise_u8
    rng = np.random.default_rng(5)
    x = rng.uniform(-0.2, 1.2, 100_000).astype(np.float32)
    x[:600] = (np.arange(600) / 2.0 / 255.0).astype(np.float32)  # halves: round-half-even territory
    want = (np.clip(x.astype(np.float64), 0.0, 1.0) * 255.0).round().astype(np.uint8)
    got = quantise_u8(torch.as_tensor(x, device="cuda")).cpu().numpy()
    np.testing.assert_array_equal(got, want)


def test_denoise_report_is_computed_on_the_device(torch_cuda, g):
    """The K6 report equals the host formulas (pipeline.py:30-51) on the returned images."""
    import importlib
    P = importlib.import_module("paper_1901_06919_b200.pipeline")
    views = _views(g)
    out, rep = P.denoise(views, P.PipelineConfig(known_shifts=_known(g)))
    # the host images are the float64 widening of the float32 renders the device compared
    host_psnr = [P.psnr(out.images[j], views.images[j]) for j in range(views.num_views)]
    np.testing.assert_allclose(rep.per_view_psnr, host_psnr, rtol=0, atol=1e-9)
    np.testing.assert_allclose(rep.per_channel_mse, P.mse_per_channel(out.images, views.images), rtol=1e-10)
    assert rep.mean_psnr == pytest.approx(float(np.mean(host_psnr)), abs=1e-9)
    assert set(rep.timings) == {"construct", "render"}
    doc = json.loads(json.dumps(rep.to_dict()))
    assert doc["per_view_psnr"] == [pytest.approx(p) for p in host_psnr]


def test_device_output_keeps_the_renders_in_hbm(torch_cuda, g):
    import importlib
    P = importlib.import_module("paper_1901_06919_b200.pipeline")
    host = P.interpolate_views(_views(g), g["targets"], P.PipelineConfig(known_shifts=_known(g)))
    dev = P.interpolate_views(_views(g), g["targets"], P.PipelineConfig(known_shifts=_known(g), device_output=True))
    assert dev.images.is_cuda and dev.images.dtype == torch_cuda.float32
    np.testing.assert_array_equal(dev.images.cpu().numpy().astype(np.float64), host.images)


def test_views_cross_pcie_once_with_calibration(torch_cuda, g, monkeypatch):
    """Calibration and construction read the SAME resident tensor (round 1 uploaded twice)."""
    import importlib
    from paper_1901_06919_b200 import CalibConfig
    Cal = importlib.import_module("paper_1901_06919_b200.calibrate")
    Con = importlib.import_module("paper_1901_06919_b200.construct")
    P = importlib.import_module("paper_1901_06919_b200.pipeline")
    seen = []
    real_spectra, real_k0 = Cal._Spectra.__init__, Con.views_to_spectra

    def spy_spectra(self, views, device=None):
        seen.append(("calibrate", views.images.is_cuda if hasattr(views.images, "is_cuda") else False))
        real_spectra(self, views, device)

    def spy_k0(views_dev, pad, srgb=False):
        seen.append(("construct", views_dev.is_cuda))
        return real_k0(views_dev, pad, srgb=srgb)

    def no_host_path(*a, **k):
        raise AssertionError("the pipeline must not re-upload the views")

    monkeypatch.setattr(Cal._Spectra, "__init__", spy_spectra)
    monkeypatch.setattr(Con, "views_to_spectra", spy_k0)
    monkeypatch.setattr(Con, "views_to_spectra_host", no_host_path)
    cal = CalibConfig(n_layers=2, batch_size=10**6, grid_dims=(3, 3), d_min=-0.2, d_max=1.2, max_iters=5, seed=0,
                      lam=1e-4)
    P.interpolate_views(_views(g), g["targets"], P.PipelineConfig(calib=cal))
    assert ("calibrate", True) in seen and ("construct", True) in seen
    assert all(on_device for _, on_device in seen)


# ---------------------------------------------------------------------------- service backend

@pytest.fixture(scope="module")
def service(torch_cuda, g):
    from paper_1901_06919_b200 import construct_fdl
    from paper_1901_06919_b200.serve import RenderService
    model = construct_fdl(_views(g, np.float32), _known(g), lam=1e-4)
    return RenderService(model, threads=2)


def _decode(body):
    from PIL import Image
    return np.asarray(Image.open(io.BytesIO(body)))


def test_info_reports_model_metadata(service, g):
    doc = service.info()
    assert doc["n"] == len(g["d"]) and len(doc["d"]) == len(g["d"])
    assert doc["width"] == g["images"].shape[2] and doc["height"] == g["images"].shape[1]
    assert "pinhole" in doc["apertures"]
    assert doc["hull"]["u"] == [float(g["coords"][:, 0].min()), float(g["coords"][:, 0].max())]


def test_png_pixels_are_the_quantised_render(service):
    from paper_1901_06919_b200 import render
    q = "u=0.25&v=-0.5&s=0.5&f=1.0&aperture=disk"
    ctype, body, ms = service.render_bytes(q)
    assert ctype == "image/png" and body[:8] == b"\x89PNG\r\n\x1a\n" and ms >= 0
    req, _, _ = service.parse_query(q)
    img = render(service.model, req)
    want = (np.clip(img, 0.0, 1.0) * 255.0).round().astype(np.uint8)  # serve.py:127 on the host
    np.testing.assert_array_equal(_decode(body), want)


def test_identical_queries_identical_bytes_and_concurrency(service):
    q = "u=0.1&v=0.1&aperture=square&f=0.5"
    a = service.render_bytes(q)[1]
    with ThreadPoolExecutor(4) as pool:
        outs = list(pool.map(lambda _: service.render_bytes("v=0.1&u=0.1")[1], range(8)))
    assert all(o == outs[0] for o in outs)
    assert service.render_bytes(q)[1] == a


def test_batched_queries_equal_single_queries(service):
    qs = [f"u={0.1 * i:.2f}&v={-0.05 * i:.2f}&f={0.25 * (i % 3)}&s=0.3" for i in range(7)]
    batch = service.render_batch_bytes(qs)
    from paper_1901_06919_b200.serve import RenderService
    fresh = RenderService(service.model, threads=1)
    for q, (ctype, body, _) in zip(qs, batch):
        assert (ctype, body) == fresh.render_bytes(q)[:2]


def test_jpeg_quality(service):
    ctype, body, _ = service.render_bytes("quality=jpeg-70")
    assert ctype == "image/jpeg" and body[:2] == b"\xff\xd8"


@pytest.mark.parametrize("query,status,needle", [
    ("f=-1", 400, "'f'"), ("u=abc", 400, "'u'"), ("aperture=octagon", 422, "octagon"),
    ("quality=bmp", 400, "quality"), ("quality=jpeg-0", 400, "1..100"), ("v=inf", 400, "finite"),
])
def test_query_errors(service, query, status, needle):
    from paper_1901_06919_b200.serve import QueryError
    with pytest.raises(QueryError) as exc:
        service.render_bytes(query)
    assert exc.value.status == status and needle in str(exc.value)

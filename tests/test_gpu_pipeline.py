"""Pipelines on the GPU (paper_1901_06919_b200.pipeline) against the reference's
outputs (tests/golden/pipeline.npz, made by tests/golden/make_pipeline.py).
Gate: rendered views >= 60 dB PSNR against the reference's (BASELINE.json)."""

import math

import numpy as np
import pytest

from conftest import load_golden, psnr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import importlib
    return importlib.import_module("paper_1901_06919_b200.pipeline")


@pytest.fixture(scope="module")
def g():
    return load_golden("pipeline")


def _views(g):
    from paper_1901_06919_b200 import ViewSet
    return ViewSet(images=g["images"], u=g["coords"][:, 0], v=g["coords"][:, 1])


def _known(g):
    from paper_1901_06919_b200 import ShiftParams
    return ShiftParams.factored(g["coords"][:, 0], g["coords"][:, 1], g["d"])


def _gate(out, ref):
    assert out.shape == ref.shape
    worst = min(psnr(out[i], ref[i]) for i in range(len(ref)))
    print(f"min PSNR vs reference {worst:.1f} dB")
    assert worst >= 60.0


def test_interpolate_known_shifts(P, g):
    sink = {}
    iv = P.interpolate_views(_views(g), g["targets"], P.PipelineConfig(known_shifts=_known(g)), report_sink=sink)
    _gate(iv.images, g["interp_known"])
    assert sink["extrapolated"] == list(g["interp_flags"])
    assert set(sink["timings"]) == {"construct", "render"}
    np.testing.assert_array_equal(iv.u, g["targets"][:, 0])


def test_interpolate_with_calibration(P, g):
    from paper_1901_06919_b200 import CalibConfig
    cal = CalibConfig(n_layers=2, batch_size=10**6, grid_dims=(3, 3), d_min=-0.2, d_max=1.2, max_iters=30, seed=0,
                      lam=1e-4)
    sink = {}
    iv = P.interpolate_views(_views(g), g["targets"], P.PipelineConfig(calib=cal), report_sink=sink)
    _gate(iv.images, g["interp_calib"])
    assert "calibrate" in sink["timings"]


def test_denoise_known_shifts(P, g):
    dn, rep = P.denoise(_views(g), P.PipelineConfig(known_shifts=_known(g)))
    _gate(dn.images, g["denoise_known"])
    np.testing.assert_allclose(rep.per_view_psnr, g["denoise_known_psnr"], atol=1e-3)
    assert rep.mean_psnr == pytest.approx(float(np.mean(g["denoise_known_psnr"])), abs=1e-3)


def test_denoise_relaxed(P, g):
    from paper_1901_06919_b200 import CalibConfig
    cal = CalibConfig(n_layers=6, batch_size=10**6, max_iters=8, seed=0, lam=1e-4)
    dr, rep = P.denoise(_views(g), P.PipelineConfig(known_shifts=_known(g), calib=cal), relaxed=True)
    _gate(dr.images, g["denoise_relaxed"])
    assert "calibrate_relaxed" in rep.timings


def test_report_and_metrics(P, tmp_path):
    a = np.zeros((4, 4, 3))
    assert P.psnr(a, a) == math.inf
    assert P.psnr(a, a + 0.1) == pytest.approx(20.0)
    assert len(P.mse_per_channel(a, a + 0.1)) == 3
    with pytest.raises(ValueError):
        P.psnr(a, np.zeros((4, 4)))
    rep = P.QualityReport(per_view_psnr=[math.inf, 30.0], mean_psnr=30.0, per_channel_mse=[0.0])
    rep.write_json(tmp_path / "r.json")
    rep.write_csv(tmp_path / "r.csv")
    assert '"inf"' in (tmp_path / "r.json").read_text()
    assert (tmp_path / "r.csv").read_text().splitlines()[1] == "0,inf"

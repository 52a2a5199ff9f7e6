"""FDL1 model files (paper_1901_06919_b200/io.py) against files written by the
reference's own save_model (tests/golden/make_fdl1.py; fdl/io.py:157-237) and
the reference's tests of the format (test_io.py:130-175,
test_acceptance.py:325-354)."""

from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture
def fdl_cpu():
    import paper_1901_06919_b200 as pkg
    return pkg


@pytest.fixture
def fdl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_06919_b200 as pkg
    return pkg


def test_reads_reference_files_and_rewrites_them_bit_exactly(fdl_cpu, tmp_path):
    from paper_1901_06919_b200.io import load_model, save_model
    for name, kind in (("ref_factored.fdl", "factored"), ("ref_relaxed.fdl", "relaxed")):
        src = GOLD / name
        model = load_model(src)
        assert model.width == 16 and model.height == 16 and model.pad_margin == 1
        assert model.layers.shape == (2, 1, 18, 10)
        assert np.array_equal(model.disparities, [0.0, 1.0])
        assert model.calibration is not None
        assert model.calibration.is_factored == (kind == "factored")
        out = tmp_path / name
        save_model(out, model)
        assert out.read_bytes() == src.read_bytes()
    relaxed = load_model(GOLD / "ref_relaxed.fdl")
    assert relaxed.lambda_used is None
    assert np.array_equal(relaxed.calibration.pu, np.outer(np.arange(9) - 4.0, [0.0, 1.0]))


def test_rejects_bad_magic_truncation_and_kind(fdl_cpu, tmp_path):
    from paper_1901_06919_b200.io import ModelFormatError, load_model
    raw = (GOLD / "ref_factored.fdl").read_bytes()
    p = tmp_path / "m.fdl"
    p.write_bytes(b"NOPE" + raw[4:])
    with pytest.raises(ModelFormatError, match="magic"):
        load_model(p)
    p.write_bytes(raw[:-11])
    with pytest.raises(ModelFormatError, match="size"):
        load_model(p)
    p.write_bytes(raw[:20])
    with pytest.raises(ModelFormatError, match="too small"):
        load_model(p)
    bad = bytearray(raw)
    bad[25] = 7  # calibration kind byte
    p.write_bytes(bytes(bad))
    with pytest.raises(ModelFormatError, match="kind"):
        load_model(p)
    assert issubclass(ModelFormatError, ValueError)


@pytest.mark.gpu
def test_device_model_round_trip(fdl, tmp_path):
    """A GPU-constructed model goes to disk from HBM and comes back into HBM
    bit-exactly; the file re-saves to identical bytes (test_io.py:130-142)."""
    import torch
    from harness.synth import make_case
    from paper_1901_06919_b200.io import load_model, save_model
    case = make_case("c1", 32)
    model = fdl.construct_fdl(fdl.ViewSet(images=case.views.numpy(), u=case.u, v=case.v),
                              fdl.ShiftParams.factored(case.u, case.v, case.d))
    p1, p2 = tmp_path / "a.fdl", tmp_path / "b.fdl"
    save_model(p1, model)
    loaded = load_model(p1)
    assert loaded.layers_device().is_cuda
    assert torch.equal(loaded.layers_device(), model.layers_device())
    save_model(p2, loaded)
    assert p1.read_bytes() == p2.read_bytes()
    assert loaded.lambda_used == model.lambda_used and loaded.calibration.is_factored
    # renders from the reloaded model are the renders of the original
    r = fdl.RenderRequest(u=1.0, v=-0.5)
    assert np.array_equal(fdl.render(loaded, r), fdl.render(model, r))

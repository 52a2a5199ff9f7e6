"""C-ABI library checks that need no GPU: it loads and exports every symbol
declared in include/fdl_b200.h; argument validation fails cleanly."""

import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "fdl_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fdl_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_symbols()
    for must in ("fdl_views_to_spectra", "fdl_solve_bins", "fdl_symmetrize", "fdl_render_spectra",
                 "fdl_spectra_to_images", "fdl_last_error"):
        assert must in names


def test_library_loads_and_exports_all_symbols():
    from paper_1901_06919_b200 import _native
    lib = _native.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _native.EXPORTS, f"{name} has no ctypes signature"
    assert lib.fdl_version() >= 100


def test_invalid_arguments_fail_without_gpu():
    from paper_1901_06919_b200 import _native
    lib = _native.lib()
    rc = lib.fdl_views_to_spectra(None, 0, 4, 4, 1, 0, None, None, None, 0, None)
    assert rc == _native.FDL_ERR_INVALID
    assert b"invalid" in lib.fdl_last_error()
    desc = _native.FdlSolveDesc()
    desc.m, desc.n, desc.C, desc.Hp, desc.Wp, desc.nrows = 2, 0, 1, 4, 4, 4
    assert lib.fdl_solve_path(desc) == _native.FDL_ERR_INVALID
    with pytest.raises(ValueError):
        _native.check(_native.FDL_ERR_INVALID, "x")


def _desc(m, n, d, u, v, ap=None):
    from paper_1901_06919_b200 import _native as nat
    keep = []
    desc = nat.FdlSolveDesc()
    desc.m, desc.n, desc.C, desc.Hp, desc.Wp, desc.nrows = m, n, 1, 8, 8, 8
    d = np.ascontiguousarray(d, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    keep += [d, u, v]
    desc.d, desc.u, desc.v = nat.dptr(d), nat.dptr(u), nat.dptr(v)
    desc.lam, desc.eps = 1.0, 1e-9
    return desc, keep


@pytest.mark.parametrize("d,u,expect", [
    (np.linspace(-1, 1, 4), [0.0, 1.0], 1),         # symmetric d, pinhole -> symmetric-real
    (np.linspace(-1, 1, 5), [0.0, 1.0], 1),         # odd n keeps the middle column
    (np.array([-1.0, 0.0, 1.0, 2.0]), [0.0, 1.0], 3),  # asymmetric d -> complex embedding
    (np.array([-1.0, 0.0, 1.0, 2.0]), [0.0, 0.0], 2),  # zero shifts -> real A
])
def test_solve_path_selection(d, u, expect):
    from paper_1901_06919_b200 import _native as nat
    desc, keep = _desc(2, len(d), d, u, [0.0, 0.0])
    assert nat.lib().fdl_solve_path(desc) == expect


def test_calibration_entry_points_validate_without_gpu():
    import ctypes
    from paper_1901_06919_b200 import _native as nat
    lib = nat.lib()
    d = nat.FdlCalibDesc()
    d.m, d.n, d.B, d.H, d.W = 2, 0, 4, 8, 8
    assert lib.fdl_calib_workspace(ctypes.byref(d)) == 0
    assert lib.fdl_calib_solve(ctypes.byref(d), None, 0, None) == nat.FDL_ERR_INVALID
    # a valid plan needs host arrays; out-of-range bins are refused before any device work
    bins = np.array([0, 1, 99], dtype=np.int32)
    pu = np.zeros((2, 2))
    gam = np.eye(2)
    d.n, d.B = 2, 3
    d.bins, d.pu, d.pv, d.gamma = nat.iptr(bins), nat.dptr(pu), nat.dptr(pu), nat.dptr(gam)
    assert lib.fdl_calib_workspace(ctypes.byref(d)) == 0
    assert b"out of range" in lib.fdl_last_error()
    bins[2] = 5
    assert lib.fdl_calib_workspace(ctypes.byref(d)) > 0
    assert lib.fdl_lstsq_minnorm_workspace(2, 3, 3, 1) > 0
    assert lib.fdl_lstsq_minnorm(-1, 3, 3, 1, None, None, None, None, None, 0, None) == nat.FDL_ERR_INVALID


def test_on_device_decorator_passes_through_without_cuda_device():
    """_native.on_device selects the CUDA device a call's tensors live on; host-only
    calls (device None or a CPU device) run untouched."""
    import torch
    from paper_1901_06919_b200 import _native as nat

    @nat.on_device(lambda x, device=None: device)
    def probe(x, device=None):
        return x + 1

    assert probe(1) == 2
    assert probe(1, device="cpu") == 2
    assert probe(1, device=torch.device("cpu")) == 2
    assert probe.__name__ == "probe"


def test_staging_arena_lifecycle_without_gpu():
    """The capture-support entry points are pure host bookkeeping until a call stages a block."""
    from paper_1901_06919_b200 import _native as nat
    L = nat.lib()
    arena = L.fdl_staging_arena_begin()
    assert arena
    assert not L.fdl_staging_arena_begin()          # one open arena per thread
    assert L.fdl_staging_arena_end(arena) == 0
    assert L.fdl_staging_arena_end(arena) != 0      # already closed
    assert L.fdl_staging_arena_free(arena) == 0


def test_quantised_images_decode_like_the_reference_loader():
    # io.py:54-59: uint8 -> / 255.0, uint16 -> / 65535.0 in float64; ViewSet keeps them quantised
    from paper_1901_06919_b200 import QuantisedImages, ViewSet
    rng = np.random.default_rng(2)
    for dtype, maxv in ((np.uint8, 255.0), (np.uint16, 65535.0)):
        q = rng.integers(0, int(maxv) + 1, (3, 5, 4, 2)).astype(dtype)
        qi = QuantisedImages(q)
        assert qi.shape == q.shape and qi.bits == 8 * np.dtype(dtype).itemsize
        assert np.array_equal(np.asarray(qi), q.astype(np.float64) / maxv)
        assert np.asarray(qi, dtype=np.float32).dtype == np.float32
        vs = ViewSet(images=qi, u=np.zeros(3), v=np.zeros(3))
        assert vs.images is qi and vs.num_views == 3 and (vs.height, vs.width, vs.channels) == (5, 4, 2)
    gray = QuantisedImages(np.zeros((2, 4, 4), np.uint8))
    assert gray.shape == (2, 4, 4, 1)
    with pytest.raises(ValueError):
        QuantisedImages(np.zeros((2, 4, 4, 1), np.float32))
    with pytest.raises(ValueError):
        QuantisedImages(np.zeros((4, 4), np.uint8))

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

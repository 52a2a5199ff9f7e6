"""The PRODUCT's aperture tables (paper_1901_06919_b200.render.aperture_spectrum)
against the reference's own tables (render.py:93-132, stored by
tests/golden/make_golden.py): the exact arrays, not the oracle's copy.

Every GPU construction / render test that builds a table with the product
function feeds it to both sides, so this is the pin for SURVEY §8(a) row r6.
"""

import numpy as np
import pytest

from conftest import load_golden
from paper_1901_06919_b200 import aperture_spectrum

HEX = [(np.cos(a), np.sin(a)) for a in np.linspace(0, 2 * np.pi, 6)[:-1]]

CASES = [
    ("c3_s32", "ap", dict(shape="disk", diameter=8.0)),
    ("render_c5_small", "ap", dict(shape="disk", diameter=1.0)),
    ("render_apertures", "poly", dict(shape="polygon", vertices=HEX, pad_factor=4)),
    ("render_apertures", "sq", dict(shape="square", side=0.5, pad_factor=4)),
]


@pytest.mark.parametrize("golden,prefix,kw", CASES, ids=[f"{c[0]}-{c[1]}" for c in CASES])
def test_product_table_equals_reference(golden, prefix, kw):
    g = load_golden(golden)
    kw = dict(kw)
    shape = kw.pop("shape")
    ap = aperture_spectrum(shape, **kw)
    ref_t = g[f"{prefix}_table"]
    assert np.iscomplexobj(ap.table) == np.iscomplexobj(ref_t)
    assert ap.table.shape == ref_t.shape
    assert np.array_equal(ap.table, ref_t), float(np.max(np.abs(ap.table - ref_t)))
    assert np.array_equal(ap.xi_x, g[f"{prefix}_xi_x"])
    assert np.array_equal(ap.xi_y, g[f"{prefix}_xi_y"])

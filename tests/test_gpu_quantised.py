"""8- / 16-bit views (the loader's on-disk format, reference io.py:54-59) through the
construction: `fdl_dequantise_views` against numpy's float64 decode on every code value,
and construct_fdl from quantised host views against the float32 decode, bit for bit."""

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


def _decode(q):
    """io.py:54-59 followed by the float32 cast of the upload."""
    maxv = 255.0 if q.dtype == np.uint8 else 65535.0
    return (q.astype(np.float64) / maxv).astype(np.float32)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
@pytest.mark.parametrize("offset", [0, 1, 3])
def test_dequantise_every_code_value(torch_cuda, dtype, offset):
    torch = torch_cuda
    from paper_1901_06919_b200 import _native as nat
    L = nat.lib()
    bits = 8 * np.dtype(dtype).itemsize
    codes = np.arange(1 << bits, dtype=dtype)
    rng = np.random.default_rng(5)
    q = np.concatenate([codes, rng.integers(0, 1 << bits, 4099).astype(dtype)])  # odd length: vector body + tail
    buf = torch.zeros(len(q) + 8, dtype=torch.uint8 if bits == 8 else torch.uint16, device="cuda")
    buf[offset:offset + len(q)].copy_(torch.from_numpy(q))
    out = torch.full((len(q) + 8,), -1.0, dtype=torch.float32, device="cuda")
    src = buf.data_ptr() + offset * np.dtype(dtype).itemsize  # offsets 1, 3: not 16-byte aligned
    nat.check(L.fdl_dequantise_views(src, bits, len(q), out[offset:].data_ptr(), nat.stream_handle(out.device)),
              "fdl_dequantise_views")
    got = out.cpu().numpy()
    assert np.array_equal(got[offset:offset + len(q)], _decode(q))
    assert np.all(got[:offset] == -1.0) and np.all(got[offset + len(q):] == -1.0)  # nothing outside the range


def test_dequantise_rejects_bad_arguments(torch_cuda):
    from paper_1901_06919_b200 import _native as nat
    L = nat.lib()
    t = torch_cuda.zeros(16, dtype=torch_cuda.float32, device="cuda")
    assert L.fdl_dequantise_views(t.data_ptr(), 12, 16, t.data_ptr(), None) == nat.FDL_ERR_INVALID
    assert L.fdl_dequantise_views(None, 8, 16, t.data_ptr(), None) == nat.FDL_ERR_INVALID
    assert L.fdl_dequantise_views(t.data_ptr(), 8, -1, t.data_ptr(), None) == nat.FDL_ERR_INVALID
    assert L.fdl_dequantise_views(None, 8, 0, None, None) == 0


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
@pytest.mark.parametrize("pinned", [False, True])
def test_construct_from_quantised_views_is_bitwise_the_float_construct(torch_cuda, dtype, pinned):
    torch = torch_cuda
    import paper_1901_06919_b200 as fdl
    g = load_golden("c2_s24")
    maxv = 255 if dtype == np.uint8 else 65535
    q = np.round(np.clip(g["views"], 0, 1) * maxv).astype(dtype)
    sh = fdl.ShiftParams.factored(g["u"], g["v"], g["d"])
    data = torch.from_numpy(q).pin_memory() if pinned else q
    qi = fdl.QuantisedImages(data)
    assert qi.shape == q.shape and qi.bits == 8 * np.dtype(dtype).itemsize
    a = fdl.construct_fdl(fdl.ViewSet(images=qi, u=g["u"], v=g["v"]), sh)
    b = fdl.construct_fdl(fdl.ViewSet(images=_decode(q), u=g["u"], v=g["v"]), sh)
    assert a.lambda_used == b.lambda_used
    assert np.array_equal(a.layers, b.layers)
    # a small upload chunk: several chunks, the decode offsets stay view-aligned
    from paper_1901_06919_b200 import construct as Cn
    sp_a, ss_a = Cn.views_to_spectra_host(qi, 3, torch.device("cuda"), chunk_bytes=5 * q[0].size * 4)
    sp_b, ss_b = Cn.views_to_spectra_host(_decode(q), 3, torch.device("cuda"))
    assert torch.equal(sp_a, sp_b) and torch.equal(ss_a, ss_b)

"""Sharded construction on the GPU (paper_1901_06919_b200/dist.py).

Only one GPU is available to the tests, so world size > 1 is emulated the
way the exchange delivers data: the row slabs of P ranks are solved one
after the other from the same spectra and must reproduce the single-GPU
layers BIT FOR BIT (per-bin arithmetic is slab-independent; the GPU analogue
of the reference's test_construct.py:196-204).  The real NCCL path runs with
world size 1 through torch.distributed.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _case(size=48):
    from harness.synth import make_case
    return make_case("c2", size, device="cuda")


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_slab_partition_bitwise(cuda, world):
    torch = cuda
    import paper_1901_06919_b200 as fdl
    from paper_1901_06919_b200 import construct as K
    from paper_1901_06919_b200 import dist as D
    case = _case()
    m, H, W, C = case.views.shape
    pu, pv = np.outer(case.u, case.d), np.outer(case.v, case.d)
    pad = K.default_pad_margin(pu, pv)
    Hp, Wp = H + 2 * pad, W + 2 * pad
    spectra, sumsq = K.views_to_spectra(case.views, pad)
    lam = K.lambda_from_sumsq(sumsq.cpu().numpy(), Hp * (Wp // 2 + 1), m)
    full, nb, _ = K.solve_slab(spectra, m, len(case.d), C, Hp, Wp, np.arange(Hp), pu, pv, case.d, lam, 1e-9,
                               u=case.u, v=case.v)
    K.symmetrize(full, Hp, Wp)
    for r in range(world):
        rows, mirror = D.slab_rows(Hp, world, r)
        idx = torch.as_tensor(rows.astype(np.int64), device="cuda")
        slab = spectra[:, :, idx].contiguous()
        lay, nb, _ = K.solve_slab(slab, m, len(case.d), C, Hp, Wp, rows, pu, pv, case.d, lam, 1e-9,
                                  u=case.u, v=case.v)
        K.symmetrize(lay, Hp, Wp, rows, mirror)
        assert torch.equal(lay, full[:, :, idx]), f"rank {r} of {world}"


def test_fft_batch_independence(cuda):
    # view-sharded K0 must give each view the same spectrum as the full batch
    torch = cuda
    from paper_1901_06919_b200 import construct as K
    case = _case()
    full, s_full = K.views_to_spectra(case.views, 12)
    part, s_part = K.views_to_spectra(case.views[10:31].contiguous(), 12)
    assert torch.equal(full[10:31], part)
    assert torch.equal(s_full[10:31], s_part)


def test_construct_sharded_world1_matches_construct_fdl(cuda):
    torch = cuda
    import torch.distributed as dist
    import paper_1901_06919_b200 as fdl
    from paper_1901_06919_b200 import dist as D
    case = _case()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sh = fdl.ShiftParams.factored(case.u, case.v, case.d)
        slab, rows, lam, pad, (Hp, Wp) = D.construct_sharded(case.views, 0, case.views.shape[0], sh)
        full = D.gather_slabs(slab, Hp)
        ref = fdl.construct_fdl(fdl.ViewSet(images=case.views, u=case.u, v=case.v), sh)
        assert lam == ref.lambda_used
        assert torch.equal(full, ref.layers_device())
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_pipelined_readback_bitwise():
    """construct_fdl from host views solves in conjugate-row slabs with the
    read-back overlapped (plane_rows = Hp, fdl_symmetrize_rows,
    fdl_rows_to_host); layers must be bit-identical to the one-launch path and
    the host copy to the device layers."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_06919_b200 as fdl
    from harness.synth import make_case
    case = make_case("c2", size=96)
    views = fdl.ViewSet(images=case.views.numpy(), u=case.u, v=case.v)
    sh = fdl.ShiftParams.factored(case.u, case.v, case.d)
    a = fdl.construct_fdl(views, sh, eager_host=True)
    b = fdl.construct_fdl(views, sh, eager_host=False)
    assert a._host_async is not None and b._host_async is None
    assert torch.equal(a.layers_device(), b.layers_device())
    assert torch.equal(a.layers_host(), b.layers_device().cpu())
    np.testing.assert_array_equal(a.layers, b.layers)


def _nccl_world1(torch):
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    return dist


@pytest.mark.parametrize("chunks", [1, 3])
def test_construct_sharded_chunked_and_fallback(cuda, chunks):
    """The chunked (overlapped) exchange + device lambda give construct_fdl's layers
    bit for bit, and a breakdown bin takes the reference's minimum-norm fallback
    (construct.py:205-210) on the sharded path as on the one-GPU path."""
    torch = cuda
    import paper_1901_06919_b200 as fdl
    from paper_1901_06919_b200 import dist as D
    from oracle import fdl_oracle as O
    dist = _nccl_world1(torch)
    try:
        case = _case()
        sh = fdl.ShiftParams.factored(case.u, case.v, case.d)
        slab, rows, lam, pad, (Hp, Wp) = D.construct_sharded(case.views, 0, case.views.shape[0], sh, chunks=chunks)
        ref = fdl.construct_fdl(fdl.ViewSet(images=case.views, u=case.u, v=case.v), sh)
        assert lam == ref.lambda_used
        assert torch.equal(D.gather_slabs(slab, Hp), ref.layers_device())
        # singular DC bin (two coincident views, eps = 0): fallback on the sharded path
        rng = np.random.default_rng(3)
        img = rng.uniform(0, 1, (2, 16, 16, 1)).astype(np.float32)
        sh2 = fdl.ShiftParams.factored([0.0, 0.0], [0.0, 0.0], [0.0, 1.0])
        slab2, _, _, _, (Hp2, _) = D.construct_sharded(torch.from_numpy(img).cuda(), 0, 2, sh2, lam=1e-3, eps=0.0,
                                                       pad_margin=0, chunks=chunks)
        one = fdl.construct_fdl(fdl.ViewSet(images=img, u=[0.0, 0.0], v=[0.0, 0.0]), sh2, lam=1e-3, eps=0.0,
                                pad_margin=0)
        assert fdl.last_construct_stats().fallback_bins >= 1
        assert torch.equal(D.gather_slabs(slab2, Hp2), one.layers_device())
        oref = O.construct(img.astype(np.float64), np.zeros((2, 2)), np.zeros((2, 2)), np.array([0.0, 1.0]),
                           lam=1e-3, eps=0.0, pad=0)
        got = D.gather_slabs(slab2, Hp2).cpu().numpy()
        assert np.linalg.norm(got - oref["layers"]) / np.linalg.norm(oref["layers"]) < 1e-6
        with pytest.raises(ValueError):
            D.construct_sharded(case.views, 0, case.views.shape[0], sh, lam=-1.0)
    finally:
        dist.destroy_process_group()

"""Multi-process host logic of the sharded construction (paper_1901_06919_b200/dist.py),
world size 2 and 3 on CPU with the gloo backend: row/view partition, the
all-to-all of spectrum rows, the view-order lambda and the slab all-gather."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_06919_b200 import dist as D


@pytest.mark.parametrize("Hp", [1, 2, 7, 8, 134, 536, 2144])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_slab_rows_partition(Hp, world):
    seen = []
    for r in range(world):
        rows, mirror = D.slab_rows(Hp, world, r)
        seen += rows.tolist()
        # mirrored pairs stay together (construct.py:286-297 stays local)
        for i, ky in enumerate(rows):
            assert rows[mirror[i]] == (Hp - ky) % Hp
    assert sorted(seen) == list(range(Hp))
    if world <= Hp // 2:
        sizes = [len(D.slab_rows(Hp, world, r)[0]) for r in range(world)]
        assert max(sizes) - min(sizes) <= 2


def test_view_range_covers():
    for m in (1, 25, 81, 289):
        for w in (1, 2, 3, 8):
            parts = [D.view_range(m, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, C, Hp, Whp, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gen = torch.Generator().manual_seed(7)
        full = torch.complex(torch.randn((m, C, Hp, Whp), generator=gen), torch.randn((m, C, Hp, Whp), generator=gen))
        j0, j1 = D.view_range(m, world, rank)
        local = full[j0:j1].contiguous()
        (slab, rows1, _), = D.exchange_rows(local, m, Hp)
        rows, _ = D.slab_rows(Hp, world, rank)
        ok_exchange = torch.equal(slab, full[:, :, torch.as_tensor(rows.astype(np.int64))])
        ok_exchange &= np.array_equal(rows1, rows)
        # the chunked (pipelined) exchange delivers the same slab, piece by piece, bit for bit
        for chunks in (2, 3, 5):
            parts = D.exchange_rows(local, m, Hp, chunks=chunks, async_op=True)
            for _, _, work in parts:
                if work is not None:
                    work.wait()
            got = torch.cat([r for r, _, _ in parts], dim=2)
            ok_exchange &= torch.equal(got, slab)
            ok_exchange &= np.array_equal(np.concatenate([rc for _, rc, _ in parts]), rows)
        # lambda from per-view partial sums: identical to the single-process value
        sums = (full.abs() ** 2).sum(dim=(1, 2, 3)).double()
        lam = D.lambda_all_views(sums[j0:j1], m, Hp * Whp)
        from paper_1901_06919_b200.construct import lambda_from_sumsq
        ok_lam = lam == lambda_from_sumsq(sums.numpy(), Hp * Whp, m)
        # slab all-gather rebuilds the full layer tensor
        layers = torch.complex(torch.randn((n, C, Hp, Whp), generator=gen), torch.randn((n, C, Hp, Whp), generator=gen))
        mine = layers[:, :, torch.as_tensor(rows.astype(np.int64))].contiguous()
        ok_gather = torch.equal(D.gather_slabs(mine, Hp), layers)
        q.put((rank, bool(ok_exchange), bool(ok_lam), bool(ok_gather)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 7), (3, 7), (3, 2)])
def test_exchange_gloo(world, m):
    # (3, 2): fewer views than ranks -- a rank with no views still takes part
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, 2, 10, 6, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert len(res) == world
    for rank, ok_x, ok_l, ok_g in res:
        assert ok_x, f"rank {rank}: all-to-all rows"
        assert ok_l, f"rank {rank}: lambda"
        assert ok_g, f"rank {rank}: slab all-gather"

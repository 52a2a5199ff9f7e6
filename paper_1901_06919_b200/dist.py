"""Multi-GPU FDL construction and rendering (one process per GPU, torch.distributed/NCCL).

Construction shards by frequency rows:

  1. views are sharded by index: rank r owns views [m r / P, m (r+1) / P) and
     runs K0 (pad + cuFFT R2C + per-view sum|b|^2) on them only;
  2. the per-view sums are all-gathered and added in view order, so lambda
     (construct.py:214-216) is bit-identical for every world size;
  3. ONE all-to-all moves every view's spectrum rows to the rank that owns
     them: rank p owns a set of mirrored row pairs {ky, Hp - ky}, so the
     self-conjugate symmetrisation (construct.py:286-297) stays local;
  4. K1 + K2 run on the local slab; layers stay slab-resident (n, C, rows, Whp).

Per-bin arithmetic does not depend on the slab, so the layers are identical
for 1, 2, 4 or 8 GPUs (the GPU analogue of test_construct.py:196-204).
Rendering replicates the layers (one all-gather) and shards the output
views; there is no exchange after that.

The row/view partition and the exchange bookkeeping are plain host logic,
tested on CPU with the gloo backend (tests/test_dist_cpu.py).
"""

from __future__ import annotations

import numpy as np

__all__ = ["row_groups", "slab_rows", "view_range", "exchange_rows", "gather_slabs", "construct_sharded",
           "lambda_all_views"]


def row_groups(Hp: int):
    """Conjugate row groups: [0], [ky, Hp - ky] for 0 < ky < Hp/2, [Hp/2] for even Hp."""
    groups = [[0]]
    for ky in range(1, (Hp + 1) // 2):
        groups.append([ky, Hp - ky])
    if Hp % 2 == 0 and Hp > 1:
        groups.append([Hp // 2])
    return groups


def slab_rows(Hp: int, world: int, rank: int):
    """(rows, mirror) of rank's slab: contiguous blocks of conjugate row groups
    balanced by row count; mirror[i] = slab index of row (Hp - rows[i]) % Hp."""
    groups = row_groups(Hp)
    sizes = np.array([len(g) for g in groups])
    cum = np.concatenate(([0], np.cumsum(sizes)))
    # group boundaries closest to equal row counts
    bounds = [0]
    for p in range(1, world):
        target = Hp * p / world
        bounds.append(int(np.argmin(np.abs(cum - target))))
    bounds.append(len(groups))
    bounds = np.maximum.accumulate(np.minimum(bounds, len(groups)))
    mine = groups[bounds[rank]:bounds[rank + 1]]
    rows = np.array(sorted(r for g in mine for r in g), dtype=np.int32)
    index = {int(r): i for i, r in enumerate(rows)}
    mirror = np.array([index[int((Hp - r) % Hp)] for r in rows], dtype=np.int32)
    return rows, mirror


def view_range(m: int, world: int, rank: int):
    """Contiguous view shard [j0, j1) of rank."""
    return (m * rank) // world, (m * (rank + 1)) // world


def lambda_all_views(local_sumsq, m: int, Q: int, group=None):
    """Default lambda from every view's sum|b|^2, added in view order (world-size independent)."""
    import torch
    import torch.distributed as dist
    from .construct import lambda_from_sumsq
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return lambda_from_sumsq(local_sumsq.cpu().numpy(), Q, m)
    per = -(-m // world)
    buf = torch.zeros(per, dtype=torch.float64, device=local_sumsq.device)
    buf[: local_sumsq.numel()] = local_sumsq
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    host = torch.cat(parts).cpu().numpy()
    ordered = np.concatenate([host[p * per: p * per + (view_range(m, world, p)[1] - view_range(m, world, p)[0])]
                              for p in range(world)])
    return lambda_from_sumsq(ordered, Q, m)


def _default_gather(src, rows):
    """(m_r, C, Hp, Whp) -> (m_r, C, len(rows), Whp) on the device via fdl_gather_rows."""
    import torch
    from . import _native as nat
    m_r, C, Hp, Whp = src.shape
    dst = torch.empty((m_r, C, len(rows), Whp), dtype=src.dtype, device=src.device)
    if dst.numel() == 0:
        return dst
    rows_dev = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.int32), device=src.device)
    nat.check(nat.lib().fdl_gather_rows(src.data_ptr(), m_r, C, Hp, Whp, rows_dev.data_ptr(), len(rows),
                                        dst.data_ptr(), nat.stream_handle(src.device)), "fdl_gather_rows")
    return dst


def exchange_rows(spectra_local, m: int, Hp: int, group=None, gather=None):
    """The all-to-all: view-sharded spectra (m_r, C, Hp, Whp) -> this rank's row slab
    of every view (m, C, nrows, Whp), views in global order."""
    import torch
    import torch.distributed as dist
    gather = gather or _default_gather
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m_r, C, _, Whp = spectra_local.shape
    slabs = [slab_rows(Hp, world, p)[0] for p in range(world)]
    send = torch.cat([gather(spectra_local, slabs[p]).reshape(-1) for p in range(world)])
    in_splits = [m_r * C * len(slabs[p]) * Whp for p in range(world)]
    counts = [view_range(m, world, s)[1] - view_range(m, world, s)[0] for s in range(world)]
    out_splits = [counts[s] * C * len(slabs[rank]) * Whp for s in range(world)]
    recv = torch.empty(sum(out_splits), dtype=spectra_local.dtype, device=spectra_local.device)
    if spectra_local.is_complex():
        # split sizes count complex elements along dim 0 of the (L, 2) real view
        dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send), out_splits, in_splits,
                               group=group)
    else:
        dist.all_to_all_single(recv, send, out_splits, in_splits, group=group)
    return recv.reshape(m, C, len(slabs[rank]), Whp)


def gather_slabs(layers_slab, Hp: int, group=None):
    """All-gather the row slabs (n, C, rows_p, Whp) into full layers (n, C, Hp, Whp) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n, C, _, Whp = layers_slab.shape
    slabs = [slab_rows(Hp, world, p)[0] for p in range(world)]
    maxr = max(len(s) for s in slabs)
    pad = torch.zeros((n, C, maxr, Whp), dtype=layers_slab.dtype, device=layers_slab.device)
    pad[:, :, : layers_slab.shape[2]] = layers_slab
    bufs = [torch.empty_like(pad) for _ in range(world)]
    if pad.is_complex():
        dist.all_gather([torch.view_as_real(b) for b in bufs], torch.view_as_real(pad), group=group)
    else:
        dist.all_gather(bufs, pad, group=group)
    full = torch.empty((n, C, Hp, Whp), dtype=layers_slab.dtype, device=layers_slab.device)
    for p in range(world):
        rows = torch.as_tensor(slabs[p].astype(np.int64), device=full.device)
        full[:, :, rows] = bufs[p][:, :, : len(slabs[p])]
    return full


def construct_sharded(views_local, view_offset: int, m: int, shifts, lam=None, eps: float = 1e-9,
                      pad_margin=None, group=None, views_meta=None, k1_events=None):
    """Frequency-slab sharded construct_fdl.

    views_local: (m_r, H, W, C) float32 CUDA tensor with this rank's views
    [view_offset, view_offset + m_r); shifts: the full ShiftParams (all m views).
    Returns (layers_slab (n, C, nrows, Whp) complex64, rows, lam, pad, (Hp, Wp)).
    """
    import torch.distributed as dist
    from . import construct as K
    from .construct import RankDeficiencyError
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    pu, pv = shifts.expand()
    n = pu.shape[1]
    d = np.asarray(shifts.d, dtype=np.float64)
    if lam == 0 and n > m:
        raise RankDeficiencyError(f"{n} layers from {m} images is ill-posed without regularization")
    if pad_margin is None:
        pad_margin = K.default_pad_margin(pu, pv)
    _, H, W, C = views_local.shape
    Hp, Wp = H + 2 * pad_margin, W + 2 * pad_margin
    Q = Hp * (Wp // 2 + 1)
    spectra, sumsq = K.views_to_spectra(views_local, pad_margin)
    if lam is None:
        lam = lambda_all_views(sumsq, m, Q, group)
    slab = exchange_rows(spectra, m, Hp, group)
    del spectra
    rows, mirror = slab_rows(Hp, world, rank)
    u = v = None
    if shifts.is_factored:
        u, v = shifts.u, shifts.v
    slab = slab.contiguous()
    if k1_events is not None:
        k1_events[0].record()
    layers, nbad, path = K.solve_slab(slab, m, n, C, Hp, Wp, rows, pu, pv, d, lam, eps,
                                      views=views_meta, u=u, v=v)
    if k1_events is not None:
        k1_events[1].record()
    if nbad:
        if lam == 0:
            raise RankDeficiencyError("singular normal matrix at some frequency")
        raise RuntimeError(f"{nbad} bins broke down in the fp64 Cholesky")
    K.symmetrize(layers, Hp, Wp, rows, mirror)
    return layers, rows, float(lam), pad_margin, (Hp, Wp)

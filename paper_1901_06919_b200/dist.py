"""Multi-GPU FDL construction and rendering (one process per GPU, torch.distributed/NCCL).

Construction shards by frequency rows:

  1. views are sharded by index: rank r owns views [m r / P, m (r+1) / P) and
     runs K0 (pad + cuFFT R2C + per-view sum|b|^2) on them only;
  2. the per-view sums are all-gathered and added in view order on the device,
     so lambda (construct.py:214-216) is bit-identical for every world size
     and K1 reads it without a host round trip;
  3. the all-to-all moves every view's spectrum rows to the rank that owns
     them (rank p owns a set of mirrored row pairs {ky, Hp - ky}, so the
     self-conjugate symmetrisation, construct.py:286-297, stays local), in
     EXCHANGE_CHUNKS asynchronous pieces: K1 solves piece c while piece c + 1
     is on NVLink;
  4. K2 runs on the local slab; layers stay slab-resident (n, C, rows, Whp).

Per-bin arithmetic does not depend on the slab, so the layers are identical
for 1, 2, 4 or 8 GPUs (the GPU analogue of test_construct.py:196-204).
Rendering replicates the layers (one all-gather) and shards the output
views; there is no exchange after that.

The row/view partition and the exchange bookkeeping are plain host logic,
tested on CPU with the gloo backend (tests/test_dist_cpu.py).
"""

from __future__ import annotations

import numpy as np

__all__ = ["row_groups", "slab_rows", "view_range", "chunk_rows", "exchange_rows", "gather_slabs",
           "construct_sharded", "lambda_all_views", "lambda_all_views_device"]


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


def _gather_views_ordered(local, m: int, group=None):
    """All-gather a per-view vector (m_r,) into the (m,) vector in view order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    per = -(-m // world)
    buf = torch.zeros(per, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    parts = torch.empty((world * per,), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(parts, buf, group=group)
    parts = parts.view(world, per)
    counts = [view_range(m, world, p)[1] - view_range(m, world, p)[0] for p in range(world)]
    return torch.cat([parts[p, :counts[p]] for p in range(world)])


def lambda_all_views(local_sumsq, m: int, Q: int, group=None):
    """Default lambda (host float) from every view's sum|b|^2, added in view order
    (world-size independent)."""
    from .construct import lambda_from_sumsq
    return lambda_from_sumsq(_gather_views_ordered(local_sumsq, m, group).cpu().numpy(), Q, m)


def lambda_all_views_device(local_sumsq, m: int, Q: int, group=None):
    """Default lambda as a (1,) float64 device tensor: the per-view sums are
    all-gathered and added in view order on the device (fdl_default_lambda), so
    K1 reads it without a host round trip; bit-identical to lambda_all_views."""
    from .construct import lambda_device
    return lambda_device(_gather_views_ordered(local_sumsq, m, group).contiguous(), Q, m)


def _default_gather(src, rows, out=None):
    """(m_r, C, Hp, Whp) -> (m_r, C, len(rows), Whp) on the device via fdl_gather_rows
    (into `out` when given: a slice of the all-to-all send buffer, no extra copy)."""
    import torch
    from . import _native as nat
    m_r, C, Hp, Whp = src.shape
    dst = out if out is not None else torch.empty((m_r, C, len(rows), Whp), dtype=src.dtype, device=src.device)
    if dst.numel() == 0:
        return dst
    rows_dev = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.int32), device=src.device)
    nat.check(nat.lib().fdl_gather_rows(src.data_ptr(), m_r, C, Hp, Whp, rows_dev.data_ptr(), len(rows),
                                        dst.data_ptr(), nat.stream_handle(src.device)), "fdl_gather_rows")
    return dst


def _torch_gather(src, rows, out=None):
    """Host fallback of _default_gather for CPU tensors (the gloo tests)."""
    import torch
    g = src[:, :, torch.as_tensor(np.asarray(rows, dtype=np.int64))]
    if out is None:
        return g
    out.copy_(g)
    return out


def chunk_rows(rows, chunks: int):
    """Split a slab's row list into `chunks` contiguous pieces (some may be empty)."""
    rows = np.asarray(rows)
    bounds = [(len(rows) * i) // chunks for i in range(chunks + 1)]
    return [rows[bounds[i]:bounds[i + 1]] for i in range(chunks)]


def exchange_rows(spectra_local, m: int, Hp: int, group=None, gather=None, chunks: int = 1, async_op: bool = False):
    """The all-to-all: view-sharded spectra (m_r, C, Hp, Whp) -> this rank's row slab
    of every view, views in global order.

    The slab rows are exchanged in `chunks` pieces (chunk c carries piece c of
    every rank's row list, chunk_rows).  Each chunk's send buffer is packed by
    one gather per peer straight into its slice (no concatenation).  Returns a
    list of (recv (m, C, rows_c, Whp), rows_c, work); with async_op the works
    are pending NCCL operations the caller waits on before using recv (so the
    solve of chunk c overlaps the exchange of chunk c + 1)."""
    import torch
    import torch.distributed as dist
    if gather is None:
        gather = _default_gather if spectra_local.is_cuda else _torch_gather
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m_r, C, _, Whp = spectra_local.shape
    slabs = [chunk_rows(slab_rows(Hp, world, p)[0], chunks) for p in range(world)]
    counts = [view_range(m, world, s)[1] - view_range(m, world, s)[0] for s in range(world)]
    out = []
    for c in range(chunks):
        in_splits = [m_r * C * len(slabs[p][c]) * Whp for p in range(world)]
        send = torch.empty(sum(in_splits), dtype=spectra_local.dtype, device=spectra_local.device)
        off = 0
        for p in range(world):
            if in_splits[p]:
                gather(spectra_local, slabs[p][c], out=send[off:off + in_splits[p]].view(m_r, C, len(slabs[p][c]), Whp))
            off += in_splits[p]
        mine = slabs[rank][c]
        out_splits = [counts[s] * C * len(mine) * Whp for s in range(world)]
        recv = torch.empty(sum(out_splits), dtype=spectra_local.dtype, device=spectra_local.device)
        if spectra_local.is_complex():
            # split sizes count complex elements along dim 0 of the (L, 2) real view
            work = dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send), out_splits, in_splits,
                                          group=group, async_op=async_op)
        else:
            work = dist.all_to_all_single(recv, send, out_splits, in_splits, group=group, async_op=async_op)
        out.append((recv.view(m, C, len(mine), Whp), mine, work))
    return out


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


EXCHANGE_CHUNKS = 4  # pieces of the all-to-all; the solve of piece c overlaps the exchange of c + 1


def construct_sharded(views_local, view_offset: int, m: int, shifts, lam=None, eps: float = 1e-9,
                      pad_margin=None, group=None, views_meta=None, k1_events=None, chunks: int = EXCHANGE_CHUNKS):
    """Frequency-slab sharded construct_fdl.

    views_local: (m_r, H, W, C) float32 CUDA tensor with this rank's views
    [view_offset, view_offset + m_r) (m_r may be 0 when there are fewer views
    than ranks); shifts: the full ShiftParams (all m views).
    Pipeline: K0 on the local views -> default lambda on the device from the
    all-gathered per-view sums -> the row exchange in `chunks` asynchronous
    all-to-alls, K1 solving chunk c while chunk c + 1 is in flight -> K2 on the
    whole slab.  Returns (layers_slab (n, C, nrows, Whp) complex64, rows, lam,
    pad, (Hp, Wp)); lam is read back (one scalar) after the slab is solved.
    """
    import torch
    import torch.distributed as dist
    from . import construct as K
    from . import _native as nat
    from .construct import RankDeficiencyError
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    pu, pv = shifts.expand()
    n = pu.shape[1]
    d = np.asarray(shifts.d, dtype=np.float64)
    if lam is not None and lam < 0:
        raise ValueError("lam must be non-negative")
    if lam == 0 and n > m:
        raise RankDeficiencyError(f"{n} layers from {m} images is ill-posed without regularization")
    if pad_margin is None:
        pad_margin = K.default_pad_margin(pu, pv)
    m_r, H, W, C = views_local.shape
    Hp, Wp = H + 2 * pad_margin, W + 2 * pad_margin
    Whp = Wp // 2 + 1
    Q = Hp * Whp
    dev = views_local.device
    if m_r:
        spectra, sumsq = K.views_to_spectra(views_local, pad_margin)
    else:  # no views on this rank: still takes part in the exchange and the lambda gather
        spectra = torch.empty((0, C, Hp, Whp), dtype=torch.complex64, device=dev)
        sumsq = torch.empty((0,), dtype=torch.float64, device=dev)
    lam_dev = lambda_all_views_device(sumsq, m, Q, group) if lam is None else None
    parts = exchange_rows(spectra, m, Hp, group, chunks=chunks, async_op=True)
    rows, mirror = slab_rows(Hp, world, rank)
    u = v = None
    if shifts.is_factored:
        u, v = shifts.u, shifts.v
    pieces, statuses, path = [], [], 1
    if k1_events is not None:
        k1_events[0].record()
    for recv, rows_c, work in parts:
        if work is not None:
            work.wait()  # the compute stream waits for this chunk only
        if len(rows_c) == 0:
            continue
        status = torch.zeros((len(rows_c), Whp), dtype=torch.int8, device=dev)
        lay, _, path = K.solve_slab(recv, m, n, C, Hp, Wp, rows_c, pu, pv, d, lam, eps, views=views_meta, u=u, v=v,
                                    status=status, count=False, lam_dev=lam_dev)
        pieces.append(lay)
        statuses.append((recv, rows_c, status))
    if k1_events is not None:
        k1_events[1].record()
    del spectra
    lam_h = float(lam_dev.item()) if lam_dev is not None else float(lam)
    # breakdown bins: the reference's minimum-norm fallback (construct.py:196-210) at its
    # granularity -- every bin of a solve chunk that holds a singular bin -- with the
    # bad-chunk sets of all ranks merged (slabs of different ranks can share a chunk)
    chunk = K.SOLVE_CHUNK
    nchunks = -(-Q // chunk)
    local = np.zeros(nchunks, dtype=np.int32)
    audited = 0
    for piece, (recv, rows_c, status) in zip(pieces, statuses):
        st = status.cpu().numpy().reshape(-1)
        suspects = np.flatnonzero(st == nat.FDL_BIN_SUSPECT)
        if suspects.size:  # the residual test itself, exactly as the 1-GPU path runs it
            _, verdicts, _ = K.solve_slab(recv, m, n, C, Hp, Wp, rows_c, pu, pv, d, lam_h, eps, views=views_meta,
                                          u=u, v=v, out=piece, status=status, audit_only=suspects)
            audited += int(np.count_nonzero(verdicts == 2))
            st = status.cpu().numpy().reshape(-1)
        bad = np.flatnonzero(st)
        if bad.size:
            gq = np.asarray(rows_c, dtype=np.int64)[bad // Whp] * Whp + bad % Whp
            local[np.unique(gq // chunk)] = 1
    flags = torch.as_tensor(local, device=dev)
    dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
    bad_chunks = np.flatnonzero(flags.cpu().numpy())
    if bad_chunks.size:
        if lam_h == 0:
            raise RankDeficiencyError("singular normal matrix at some frequency")
        for piece, (recv, rows_c, status) in zip(pieces, statuses):
            bins = K.fallback_bins(np.zeros(len(rows_c) * Whp, np.int8), rows_c, Whp, chunk,
                                   chunk_sync=lambda _c: bad_chunks)
            if bins.size:
                K.solve_slab(recv, m, n, C, Hp, Wp, rows_c, pu, pv, d, lam_h, eps, views=views_meta, u=u, v=v,
                             out=piece, status=status, resolve_only=bins)
                left = int(torch.count_nonzero(status).item())
                if left:
                    raise nat.FdlNativeError(f"{left} bins could not be solved (minimum-norm fallback failed)")
    layers = torch.cat(pieces, dim=2) if len(pieces) != 1 else pieces[0]
    K.symmetrize(layers, Hp, Wp, rows, mirror)
    return layers, rows, lam_h, pad_margin, (Hp, Wp)

"""Where the end-to-end construction time goes (C2): H2D alone, construct from
host views (overlapped upload + read-back), from device views with and without
the overlapped read-back."""
import time

import numpy as np
import torch

import paper_1901_06919_b200 as fdl
from harness.synth import make_case

case = make_case("c2", device="cuda")
host = torch.empty(tuple(case.views.shape), dtype=torch.float32, pin_memory=True)
host.copy_(case.views.cpu())
dev = case.views.contiguous()
sh = fdl.ShiftParams.factored(case.u, case.v, case.d)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


buf = torch.empty_like(dev)
print("H2D 255 MB pinned      %.2f ms" % timeit(lambda: buf.copy_(host, non_blocking=True)))
lay = fdl.construct_fdl(fdl.ViewSet(images=dev, u=case.u, v=case.v), sh).layers_device()
hl = torch.empty(lay.shape, dtype=lay.dtype, pin_memory=True)
print("D2H layers %.0f MB      %.2f ms" % (lay.numel() * 8 / 1e6, timeit(lambda: hl.copy_(lay, non_blocking=True))))
vh = fdl.ViewSet(images=host, u=case.u, v=case.v)
vd = fdl.ViewSet(images=dev, u=case.u, v=case.v)
print("construct host, eager  %.2f ms" % timeit(lambda: fdl.construct_fdl(vh, sh).layers_host()))
print("construct host, plain  %.2f ms" % timeit(lambda: fdl.construct_fdl(vh, sh, eager_host=False).layers_host()))
print("construct dev, eager   %.2f ms" % timeit(lambda: fdl.construct_fdl(vd, sh, eager_host=True).layers_host()))
print("construct dev, plain   %.2f ms" % timeit(lambda: fdl.construct_fdl(vd, sh, eager_host=False)))
print("construct dev, plain+D2H %.2f ms" % timeit(lambda: fdl.construct_fdl(vd, sh, eager_host=False).layers_host()))

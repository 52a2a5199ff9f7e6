"""K1 occupancy probe: a C4-like system (n = 64 layers, mirror-pair split, 8 blocks) on 9 x 9 views of
1024^2, whose per-warp shared memory (phase-table column of 9 distinct u, 243-plane tile) lets 12 warps
fit next to the default 8.  Prints the K1 kernel time per launch (library kernel timer)."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1901_06919_b200 as fdl  # noqa: E402
from harness.synth import make_case  # noqa: E402
from paper_1901_06919_b200 import _native as nat  # noqa: E402

case = make_case("c4", size=int(sys.argv[1]) if len(sys.argv) > 1 else 1024, device="cuda", side=9)
views = fdl.ViewSet(images=case.views, u=case.u, v=case.v)
sh = fdl.ShiftParams.factored(case.u, case.v, case.d)
L = nat.lib()
for _ in range(2):
    fdl.construct_fdl(views, sh)
torch.cuda.synchronize()
L.fdl_kernel_timer(1)
steps = 5
for _ in range(steps):
    model = fdl.construct_fdl(views, sh)
torch.cuda.synchronize()
tot, cnt = ctypes.c_double(0.0), ctypes.c_int32(0)
nat.check(L.fdl_kernel_timer_read(0, ctypes.byref(tot), ctypes.byref(cnt)), "timer")
L.fdl_kernel_timer(0)
st = fdl.last_construct_stats()
print(f"K1 path {st.path}: {tot.value / max(1, cnt.value):.3f} ms per launch ({cnt.value} launches), "
      f"grid {model.grid.height}x{model.grid.width}, m={len(case.u)}, n={len(case.d)}")

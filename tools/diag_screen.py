"""Residual-screen diagnostics: audited / re-solved bins and construct time per config."""
import sys, time
import numpy as np, torch
import paper_1901_06919_b200 as fdl
from harness.synth import make_case

for name in sys.argv[1:] or ["c1", "c2", "c3"]:
    case = make_case(name, device="cuda")
    views = fdl.ViewSet(images=case.views, u=case.u, v=case.v, s=getattr(case, "s", None),
                        apertures=getattr(case, "apertures", None), aperture_scale=getattr(case, "aperture_scale", None))
    sh = fdl.ShiftParams.factored(case.u, case.v, case.d)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        model = fdl.construct_fdl(views, sh)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    st = fdl.last_construct_stats()
    print(f"{name}: construct {dt*1e3:.2f} ms, audited {st.audited_bins}, re-solved {st.fallback_bins}, breakdown {st.breakdown_bins}", flush=True)

"""One small pass through every hot kernel for compute-sanitizer (memcheck / racecheck):
C1-style construct + render (K0, K1, K2, K3 Horner, K4 engine), an aperture batch (factor
pre-pass + TMA aperture tile), a relaxed-shift render (direct pinhole tile), the residual
audit path and one 1920 x 1080 K4 on the mixed-radix engine."""
import importlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1901_06919_b200 as fdl
from harness.synth import make_case

R = importlib.import_module("paper_1901_06919_b200.render")
size = int(sys.argv[1]) if len(sys.argv) > 1 else 32
case = make_case("c1", size)
views = fdl.ViewSet(images=case.views.numpy(), u=case.u, v=case.v)
sh = fdl.ShiftParams.factored(case.u, case.v, case.d)
model = fdl.construct_fdl(views, sh)
imgs = fdl.render_many(model, [fdl.RenderRequest(u=0.5, v=-0.25), fdl.RenderRequest(u=-1.0, v=1.0)])
ap = fdl.aperture_spectrum("disk", diameter=1.0)
imgs += fdl.render_many(model, [fdl.RenderRequest(u=0.2, v=0.1, s=0.3, f=1.5, aperture=ap),
                                fdl.RenderRequest(u=-0.2, v=0.4, s=-0.5, f=0.7, aperture=ap)])
pu, pv = sh.expand()
relaxed = fdl.ShiftParams.relaxed(pu + 0.01 * np.sin(np.arange(pu.size)).reshape(pu.shape), pv, d=case.d)
out = fdl.render_views_with_shifts(model, relaxed)
# residual screen + audit (tests/golden/residfire.npz when present)
try:
    g = np.load("tests/golden/residfire.npz")
    fdl.construct_fdl(fdl.ViewSet(images=g["views"], u=g["u"], v=g["v"]), fdl.ShiftParams.factored(g["u"], g["v"], g["d"]),
                      lam=float(g["lam"]), eps=float(g["eps"]))
    print("audited", fdl.last_construct_stats().audited_bins)
except FileNotFoundError:
    pass
if len(sys.argv) > 2:
    spec = torch.randn(1, 3, 1080, 961, dtype=torch.complex64, device="cuda")
    R.spectra_to_images(spec, 1080, 1920, 0, 1080, 1920)
torch.cuda.synchronize()
print("ok", len(imgs), out.shape, float(np.abs(imgs[0]).mean()))

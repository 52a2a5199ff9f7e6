"""Residual-screen diagnostics: audited / re-solved bins and K1 stage time per config (bench.py's construct path)."""
import sys, time
sys.path.insert(0, ".")
import importlib
import numpy as np, torch
import paper_1901_06919_b200 as fdl
K = importlib.import_module("paper_1901_06919_b200.construct")
import bench

for name in sys.argv[1:] or ["c1", "c2", "c3"]:
    case = bench.make_workload(name, None, torch.device("cuda"))
    views = case.views
    m, H, W, C = views.shape
    d, u, v = case.d, case.u, case.v
    n = len(d)
    wide = case.aperture is not None
    ap = fdl.aperture_spectrum(case.aperture["shape"], diameter=case.aperture["diameter"]) if wide else None
    vs_meta = fdl.ViewSet(images=np.zeros((m, 1, 1, C), np.float32), u=u, v=v, s=case.s,
                          apertures=[ap] * m if wide else None)
    pu, pv = np.outer(u, d), np.outer(v, d)
    pad = K.default_pad_margin(pu, pv)
    Hp, Wp = H + 2 * pad, W + 2 * pad
    Q = Hp * (Wp // 2 + 1)
    for rep in range(3):
        spectra, sumsq = K.views_to_spectra(views, pad)
        lam_dev = K.lambda_device(sumsq, Q, m)
        K.last_construct_stats().audited_bins = 0
        torch.cuda.synchronize(); t0 = time.perf_counter()
        layers, nbad, path = K.solve_slab(spectra, m, n, C, Hp, Wp, np.arange(Hp), pu, pv, d, None, K.DEFAULT_EPS,
                                          views=vs_meta, u=None if wide else u, v=None if wide else v, lam_dev=lam_dev)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    st = K.last_construct_stats()
    print(f"{name}: K1 stage {dt*1e3:.2f} ms, path {path}, audited {st.audited_bins}, re-solved {st.fallback_bins}, bad {nbad}", flush=True)

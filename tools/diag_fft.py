"""Diagnostic: isolate the spectra precision (cuFFT fp32 vs exact fp64 rounded to c64)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import load_golden, rel_l2
from paper_1901_06919_b200 import construct as K
from oracle import fdl_oracle as O

for name in sys.argv[1:] or ["c2_s24"]:
    g = load_golden(name)
    pad = int(g["pad"]); lam = float(g["lam"])
    m, n = len(g["u"]), len(g["d"])
    views = np.asarray(g["views"])
    if views.ndim == 3:
        views = views[..., None]
    C = views.shape[3]
    hp, wp = views.shape[1] + 2 * pad, views.shape[2] + 2 * pad
    whp = wp // 2 + 1
    spec_gpu, _ = K.views_to_spectra(torch.from_numpy(np.ascontiguousarray(views)).cuda(), pad)
    b_all, _, _ = O.view_spectra(views, pad)  # (Q, m, C) exact fp64
    spec_np = b_all.transpose(1, 2, 0).reshape(m, C, hp, whp)
    d_fft = np.abs(spec_gpu.cpu().numpy() - spec_np.astype(np.complex64))
    print(name, "max |cuFFT - fp64| / max|b|:", d_fft.max() / np.abs(spec_np).max(),
          "median rel:", np.median(d_fft / (np.abs(spec_np) + 1e-30)))
    for label, spec in [("cufft32", spec_gpu), ("exact->c64", torch.from_numpy(spec_np.astype(np.complex64)).cuda())]:
        L, nb, path = K.solve_slab(spec.contiguous(), m, n, C, hp, wp, np.arange(hp), None, None, g["d"], lam, 1e-9,
                                   u=g["u"], v=g["v"])
        K.symmetrize(L, hp, wp)
        print(f"  {label}: path {path} err {rel_l2(L.cpu().numpy(), g['layers']):.3e}")

"""Diagnostic: per-path layer error vs the golden reference, worst bins."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import load_golden, rel_l2
import paper_1901_06919_b200 as fdl

for name in sys.argv[1:] or ["c2_s24", "c1_full", "c3_s32"]:
    g = load_golden(name)
    m = len(g["u"])
    ap = None
    if "ap_table" in g:
        ap = fdl.ApertureSpec(shape="g", pad_factor=4, table=g["ap_table"], xi_x=g["ap_xi_x"], xi_y=g["ap_xi_y"])
    views = fdl.ViewSet(images=g["views"], u=g["u"], v=g["v"], s=g["s"], apertures=[ap] * m if ap else None)
    lam = None if np.isnan(g["lam_in"]) else float(g["lam_in"])
    pad = None if int(g["pad_in"]) < 0 else int(g["pad_in"])
    sh = fdl.ShiftParams.factored(g["u"], g["v"], g["d"])
    for fp in (0, 3):
        try:
            mdl = fdl.construct_fdl(views, sh, lam=lam, pad_margin=pad, force_path=fp)
        except Exception as e:
            print(name, fp, "ERR", e); continue
        L = mdl.layers
        ref = g["layers"]
        err = rel_l2(L, ref)
        per = np.linalg.norm((L - ref).reshape(L.shape[0] * L.shape[1], -1), axis=0)
        top = np.argsort(per)[::-1][:4]
        whp = L.shape[3]
        print(f"{name} path={fdl.last_construct_stats().path} err={err:.3e} floor={g['floor']} lam={mdl.lambda_used:.6g}/{float(g['lam']):.6g}",
              [(int(t % whp), int(t // whp), float(per[t])) for t in top])

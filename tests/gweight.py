"""G-weighted relative layer error — test helper.

    err_G = sqrt( sum_q (x_q - r_q)^H G_q (x_q - r_q) / sum_q r_q^H G_q r_q ),
    G_q = A_q^H A_q + lam diag(reg_q)          (construct.py:183-197)

summed over bins q and channels.  Unlike plain relative L2 it is well posed
on ill-conditioned bins (two correct fp64 solvers agree to <= 5e-6 in it,
SURVEY.md Appendix A), so it gates the fixtures whose plain-L2 floor is large.
(x - r)^H G (x - r) = ||A (x - r)||^2 + lam sum_k reg_k |x_k - r_k|^2 is
evaluated with the oracle's A (oracle/fdl_oracle.py:system_block).
"""

import numpy as np

from oracle import fdl_oracle as O


def g_weighted_error(layers, ref, u, v, d, lam, hp, wp, pu=None, pv=None, views_ap=None, eps=O.DEFAULT_EPS,
                     chunk=4096):
    layers = np.asarray(layers, dtype=np.complex128)
    ref = np.asarray(ref, dtype=np.complex128)
    n, C, _, whp = ref.shape
    if pu is None:
        pu, pv = np.outer(u, d), np.outer(v, d)
    m = pu.shape[0]
    if views_ap is None:
        views_ap = [(None, 0.0, 1.0)] * m
    px, py = O.axis_phases(pu, pv, wp, hp)
    ox, oy = O.omega_axes(wp, hp)
    e_all = (layers - ref).reshape(n, C, hp * whp).transpose(2, 0, 1)
    r_all = ref.reshape(n, C, hp * whp).transpose(2, 0, 1)
    num = den = 0.0
    for q0 in range(0, hp * whp, chunk):
        q = np.arange(q0, min(q0 + chunk, hp * whp))
        kx, ky = q % whp, q // whp
        A = O.system_block(px, py, kx, ky, d, views_ap, ox, oy)
        reg = (ox[kx] ** 2 + oy[ky] ** 2)[:, None] ** 2 * (np.asarray(d) ** 4)[None, :] + eps
        for vec, acc in ((e_all[q], "num"), (r_all[q], "den")):
            val = float(np.sum(np.abs(A @ vec) ** 2) + lam * np.sum(reg[:, :, None] * np.abs(vec) ** 2))
            if acc == "num":
                num += val
            else:
                den += val
    return float(np.sqrt(num / den))

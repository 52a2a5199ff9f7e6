"""K0 / K4 alone at a config's grid: views (m, S, S, 3) -> spectra -> images, GB/s of algorithmic traffic."""
import importlib, sys
import torch
sys.path.insert(0, ".")
K = importlib.import_module("paper_1901_06919_b200.construct")
R = importlib.import_module("paper_1901_06919_b200.render")

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
pad = int(sys.argv[2]) if len(sys.argv) > 2 else 48
m = int(sys.argv[3]) if len(sys.argv) > 3 else 48
C = 3
views = torch.rand(m, S, S, C, device="cuda")
Hp = Wp = S + 2 * pad

def timed(fn, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)

spec = [None]
def k0():
    spec[0], _ = K.views_to_spectra(views, pad)
t0 = timed(k0)
gb0 = (views.numel() * 4 + spec[0].numel() * 8) / 1e9
print(f"K0 {S}+2*{pad}, {m} views: {t0:.3f} ms, {gb0 / t0 * 1e3:.0f} GB/s algorithmic ({t0 * 289 / m:.1f} ms per 289 views)")
s = spec[0]
def k4():
    R.spectra_to_images(s, Hp, Wp, pad, S, S)
t4 = timed(k4)
print(f"K4: {t4:.3f} ms, {gb0 / t4 * 1e3:.0f} GB/s algorithmic ({t4 * 289 / m:.1f} ms per 289 views)")

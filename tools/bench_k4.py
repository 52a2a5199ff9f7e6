"""K4 alone on a config-5 sized batch: spectra (V, 3, 1080, 961) -> images, engine vs forced cuFFT."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1901_06919_b200 import _native
import importlib
R = importlib.import_module("paper_1901_06919_b200.render")

V = int(sys.argv[1]) if len(sys.argv) > 1 else 256
Hp, Wp, C = 1080, 1920, 3
spec = torch.randn(V, C, Hp, Wp // 2 + 1, dtype=torch.complex64, device="cuda")
lib = _native.lib()
for mode in ("engine", "cufft"):
    lib.fdl_fft_force_cufft(1 if mode == "cufft" else 0)
    for _ in range(2):
        R.spectra_to_images(spec.clone(), Hp, Wp, 0, Hp, Wp)
    ts = []
    for _ in range(5):
        s = spec.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        R.spectra_to_images(s, Hp, Wp, 0, Hp, Wp)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    gb = (V * C * Hp * (Wp // 2 + 1) * 8 + V * C * Hp * Wp * 4) / 1e9
    print(f"{mode}: {min(ts):.3f} ms per {V} views ({gb / min(ts) * 1e3:.0f} GB/s algorithmic)")
lib.fdl_fft_force_cufft(0)

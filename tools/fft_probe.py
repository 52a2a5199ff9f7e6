"""Probe cuFFT variants for the awkward padded sizes (536 = 8*67, 1048 = 8*131, 2144 = 32*67)."""
import torch, time
def bench(fn, x, it=10):
    for _ in range(3): fn(x)
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn(x)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/it
for (planes, n) in [(243, 536), (243, 1048), (60, 2144), (243, 512), (243, 540), (243, 544)]:
    x = torch.rand(planes, n, n, device="cuda")
    t2d = bench(lambda a: torch.fft.rfft2(a), x)
    t1d = bench(lambda a: torch.fft.fft(torch.fft.rfft(a, dim=-1), dim=-2), x)
    gb = planes * n * n * 4 * 3 / 1e9
    print(f"{planes} x {n}^2: rfft2 {t2d:.3f} ms, rfft+fft {t1d:.3f} ms, HBM-bound ~{gb/6.5:.3f} ms")

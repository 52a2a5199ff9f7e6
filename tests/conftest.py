import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def golden_aperture(g, prefix):
    """ApertureSpec-like triple stored by make_golden.py, or None."""
    if f"{prefix}_table" not in g:
        return None
    return g[f"{prefix}_table"], g[f"{prefix}_xi_x"], g[f"{prefix}_xi_y"]


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def psnr(a, b, peak=None):
    """PSNR in dB of a against the reference b (peak: b's dynamic range, >= 1)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    mse = float(np.mean((a - b) ** 2))
    if peak is None:
        peak = max(1.0, float(b.max() - b.min()))
    if mse == 0:
        return float("inf")
    return 10 * np.log10(peak ** 2 / mse)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)

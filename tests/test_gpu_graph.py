"""CUDA-graph replay of construction + renders (paper_1901_06919_b200/graph.py) against the
eager path: same kernels, same order, so layers and images must be bit-identical."""

import importlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1901_06919_b200 as fdl
    G = importlib.import_module("paper_1901_06919_b200.graph")
    R = importlib.import_module("paper_1901_06919_b200.render")
    return torch, fdl, G, R


def _rig(fdl, rng, size=64, side=3, n=6, C=1):
    g = np.arange(side) - (side - 1) / 2
    u = np.array([a for b in g for a in g], dtype=np.float64)
    v = np.array([b for b in g for a in g], dtype=np.float64)
    d = np.linspace(-1.5, 1.5, n)
    frames = [rng.uniform(0, 1, (side * side, size, size, C)).astype(np.float32) for _ in range(3)]
    return u, v, d, frames


@pytest.mark.parametrize("C,wide", [(1, False), (3, True)])
def test_graph_replay_equals_eager(env, C, wide):
    torch, fdl, G, R = env
    rng = np.random.default_rng(11 + C)
    u, v, d, frames = _rig(fdl, rng, C=C)
    shifts = fdl.ShiftParams.factored(u, v, d)
    ap = fdl.aperture_spectrum("disk", diameter=1.0)
    reqs = [fdl.RenderRequest(u=0.4 * i - 1, v=0.3 * i - 0.8, s=0.1 * i, f=(0.4 * i if wide else 0.0), aperture=ap)
            for i in range(7)]
    g = G.GraphedConstruct(fdl.ViewSet(images=frames[0], u=u, v=v), shifts, requests=reqs)
    for frame in frames[1:] + frames[:1]:
        model, images = g(frame)
        g.check()
        dev = torch.from_numpy(frame).cuda()
        eager = fdl.construct_fdl(fdl.ViewSet(images=dev, u=u, v=v), shifts)
        assert torch.equal(model.layers_device(), eager.layers_device())
        assert model.lambda_used == eager.lambda_used
        eager_imgs, _ = R.render_many_device(eager, reqs, batch=64)
        assert torch.equal(images, eager_imgs)


def test_graph_reports_bins_that_need_the_fallback(env):
    torch, fdl, G, R = env
    from conftest import load_golden
    g = load_golden("nearsingular")  # the DC bin's normal matrix is exactly singular
    views = fdl.ViewSet(images=g["views"], u=g["u"], v=g["v"])
    shifts = fdl.ShiftParams.factored(g["u"], g["v"], g["d"])
    gc = G.GraphedConstruct(views, shifts, lam=float(g["lam"]), eps=float(g["eps"]))
    gc()
    from paper_1901_06919_b200._native import FdlNativeError
    with pytest.raises(FdlNativeError, match="fallback"):
        gc.check()

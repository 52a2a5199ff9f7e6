"""Out-of-bounds write detection without compute-sanitizer (closed on this GPU pool,
profiles/r02_sanitizer.txt): every CUDA buffer the host layer allocates while a hot path
runs -- outputs, intermediates and the workspaces handed to the C ABI -- is carved out of
a larger arena whose margins hold a canary pattern; after the call the margins must be
intact.  Shapes are chosen ragged (views not a multiple of the views-per-CTA, grids not a
multiple of the bin tile, odd grids) so that every kernel's edge handling is exercised."""

import contextlib
import importlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes on each side
CANARY = 0xA5


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@contextlib.contextmanager
def guarded_allocations(torch):
    """Patch torch.empty / torch.zeros so CUDA allocations sit between canary margins."""
    arenas = []
    real_empty, real_zeros = torch.empty, torch.zeros

    def carve(shape, dtype, device, fill_zero):
        dtype = dtype or torch.get_default_dtype()
        shape = tuple(shape[0]) if len(shape) == 1 and isinstance(shape[0], (tuple, list, torch.Size)) else tuple(shape)
        nbytes = int(np.prod(shape, dtype=np.int64)) * torch.empty((), dtype=dtype).element_size()
        pad = (-nbytes) % 16
        arena = torch.full((GUARD + nbytes + pad + GUARD,), CANARY, dtype=torch.uint8, device=device)
        arenas.append((arena, nbytes + pad))
        inner = arena[GUARD:GUARD + nbytes]
        if fill_zero:
            inner.zero_()
        return inner.view(dtype).view(shape) if nbytes else real_empty(shape, dtype=dtype, device=device)

    def is_cuda(device):
        return device is not None and torch.device(device).type == "cuda"

    def empty(*shape, dtype=None, device=None, pin_memory=False, **kw):
        if is_cuda(device) and not pin_memory and not kw:
            return carve(shape, dtype, device, False)
        return real_empty(*shape, dtype=dtype, device=device, pin_memory=pin_memory, **kw)

    def zeros(*shape, dtype=None, device=None, **kw):
        if is_cuda(device) and not kw:
            return carve(shape, dtype, device, True)
        return real_zeros(*shape, dtype=dtype, device=device, **kw)

    torch.empty, torch.zeros = empty, zeros
    try:
        yield arenas
    finally:
        torch.empty, torch.zeros = real_empty, real_zeros


def assert_margins_intact(torch, arenas):
    torch.cuda.synchronize()
    assert arenas, "no guarded allocation was made"
    for arena, n in arenas:
        head, tail = arena[:GUARD], arena[GUARD + n:]
        assert bool((head == CANARY).all()), "write before the start of a device buffer"
        assert bool((tail == CANARY).all()), "write past the end of a device buffer"


def _case(fdl, size, n_layers, side, C, seed):
    rng = np.random.default_rng(seed)
    g = (np.arange(side) - (side - 1) / 2)
    u = np.array([a for b in g for a in g], dtype=np.float64)
    v = np.array([b for b in g for a in g], dtype=np.float64)
    d = np.linspace(-1.5, 1.5, n_layers)
    views = rng.uniform(0, 1, (side * side, size[0], size[1], C)).astype(np.float32)
    return fdl.ViewSet(images=views, u=u, v=v), fdl.ShiftParams.factored(u, v, d), d


@pytest.mark.parametrize("size,n_layers,C", [((128, 128), 12, 1), ((40, 52), 7, 3), ((33, 31), 5, 2)])
def test_construct_and_renders_stay_inside_their_buffers(torch_cuda, size, n_layers, C):
    torch = torch_cuda
    import paper_1901_06919_b200 as fdl
    views, shifts, d = _case(fdl, size, n_layers, 3, C, seed=size[0])
    ap = fdl.aperture_spectrum("disk", diameter=1.0)
    sq = fdl.aperture_spectrum("square", side=1.0)
    with guarded_allocations(torch) as arenas:
        model = fdl.construct_fdl(views, shifts)                      # K0 (engine or cuFFT), K1, screen, K2
        reqs = [fdl.RenderRequest(u=0.3 * i - 1.0, v=0.2 * i - 0.7) for i in range(11)]      # Horner tile + K4
        fdl.render_many(model, reqs)
        reqs = [fdl.RenderRequest(u=0.1 * i, v=-0.1 * i, s=0.2 * i - 1, f=0.5 + 0.3 * i, aperture=ap if i % 3 else sq)
                for i in range(13)]                                                          # affine aperture tile
        fdl.render_many(model, reqs)
        pu, pv = shifts.expand()
        wobble = 0.01 * np.sin(np.arange(pu.size)).reshape(pu.shape)
        relaxed = fdl.ShiftParams.relaxed(pu + wobble, pv - wobble, d=d)
        fdl.render_views_with_shifts(model, relaxed)                                         # direct pinhole tile
        assert_margins_intact(torch, arenas)


def test_relaxed_aperture_batch_and_complex_table(torch_cuda):
    """The TMA tile with 16-byte factors (non-affine shifts) and the generic tile (complex table)."""
    torch = torch_cuda
    import paper_1901_06919_b200 as fdl
    R = importlib.import_module("paper_1901_06919_b200.render")
    views, shifts, d = _case(fdl, (36, 44), 9, 3, 3, seed=5)
    model = fdl.construct_fdl(views, shifts)
    layers = model.layers_device()
    Hp, Wp = model.grid.height, model.grid.width
    ap = fdl.aperture_spectrum("disk", diameter=1.0)
    apc = fdl.ApertureSpec(shape="c", pad_factor=ap.pad_factor, table=np.asarray(ap.table).astype(np.complex128),
                           xi_x=ap.xi_x, xi_y=ap.xi_y)
    V, n = 11, len(d)
    rng = np.random.default_rng(0)
    pu = rng.uniform(-2, 2, (V, n))  # not affine in the layer index
    pv = rng.uniform(-2, 2, (V, n))
    t = rng.uniform(-3, 3, (V, n))
    with guarded_allocations(torch) as arenas:
        for table in (ap, apc):
            oob = torch.zeros((V,), dtype=torch.int64, device=layers.device)
            R.render_spectra_batch(layers, d, Hp, Wp, pu, pv, t=t, view_ap=np.zeros(V, np.int32), apertures=[table],
                                   oob=oob)
        assert_margins_intact(torch, arenas)


@pytest.mark.parametrize("V,C,Hp,Wp,pad", [(1, 3, 1080, 1920, 0), (2, 1, 1920, 1080, 3), (3, 2, 268, 134, 5),
                                           (2, 3, 50, 46, 2)])
def test_k4_stays_inside_its_buffers(torch_cuda, V, C, Hp, Wp, pad):
    torch = torch_cuda
    R = importlib.import_module("paper_1901_06919_b200.render")
    spec = torch.randn(V, C, Hp, Wp // 2 + 1, dtype=torch.complex64, device="cuda")
    with guarded_allocations(torch) as arenas:
        R.spectra_to_images(spec, Hp, Wp, pad, Hp - 2 * pad, Wp - 2 * pad)
        assert_margins_intact(torch, arenas)


def test_pipeline_report_and_quantiser(torch_cuda):
    torch = torch_cuda
    import paper_1901_06919_b200 as fdl
    P = importlib.import_module("paper_1901_06919_b200.pipeline")
    S = importlib.import_module("paper_1901_06919_b200.serve")
    views, shifts, d = _case(fdl, (30, 34), 4, 3, 3, seed=9)
    with guarded_allocations(torch) as arenas:
        out, rep = P.denoise(views, P.PipelineConfig(known_shifts=shifts, device_output=True))
        S.quantise_u8(out.images)
        assert_margins_intact(torch, arenas)
    assert len(rep.per_view_psnr) == 9

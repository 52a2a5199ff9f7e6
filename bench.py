"""Benchmark of the FDL construction + rendering hot paths (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config headline] [--impl ours|reference]

Default workload ("headline", BASELINE.json's metric "FDL construction
freq·layers/s and rendered views/s at 1/2/4/8 B200 vs roofline"):

* construction: config 4 (BASELINE.json configs[3]) — 289 views 17x17,
  2048x2048 RGB float32, 64 layers d = linspace(-6, 6, 64), pad 48 -> a
  2144 x 2144 grid, Q = 2,300,512 frequency bins.  One step = K0 (pad + R2C
  + per-view sum|b|^2) -> default lambda -> K1 (per-bin fp64 solve) -> K2
  (symmetrisation).  `value` = Q n / t (freq·layers/s).
* rendering: config 5 (configs[4]) — a 64-layer 1920x1080 RGB FDL, 4096
  requests with u, v ~ U[-4, 4], s ~ U[-5, 5], disk aperture radius
  r ~ U[0, 3] (f = 2r through one disk(1) table).  One step = all 4096 views
  (K3 weighted layer sum + K4 inverse FFT / crop) in 256-view launches.
  `render.value` = views/s.

Inputs are resident in HBM when the timed region starts and exceed the
126 MB L2 (C4 views 14.5 GB, C5 layers 1.59 GB), so no explicit flush is
needed.  `e2e` times the same work through the public API from pinned host
buffers (construct_fdl from host views, layers read back; render_many
returning float64 host images like the reference).  Other workloads:
--config c1 | c2 | c2b | c3 | c4 | c5 | calib.

Multi-GPU (torchrun, one process per GPU, NCCL): construction shards views
for K0, exchanges spectrum rows with one all-to-all and solves a frequency-row
slab per rank (paper_1901_06919_b200/dist.py); rendering shards the 4096
views.  Total work is fixed (`scaling: strong`); times are max over ranks.

--impl reference times the reference's CPU algorithm (the oracle port,
oracle/fdl_oracle.py, pinned bit-exactly to the reference's outputs) on the
host cores on bounded samples of the same workloads (same seeded inputs):
see `c4_cpu_sample` / `c5_cpu_sample`.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FDL construction freq·layers/s and rendered views/s"
FP64_PEAK_TFLOPS = 36.88  # DMMA m8n8k4 measured on this pool's B200 (profiles/r01_fp64_pipes.txt)
FP32_PEAK_TFLOPS = 73.45  # FFMA2 (fma.rn.f32x2) measured on this pool's B200 (profiles/r01_fp32_pipes.txt)
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
TRAFFIC_FILE = ROOT / "profiles" / "k1_traffic.json"  # dram bytes per K1 launch from `ncu --set full`
C5_VIEWS = 4096
C5_BATCH = 256


def hbm_peak():
    try:
        return float(json.load(open(PEAKS_FILE))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (of measured)"
    except Exception:
        return HBM_FALLBACK_GBS, "B200_PROFILING.md fallback (of fallback)"


def hbm_roofline(kernel: str, bytes_per_step: float, s_per_step: float, note: str = "", traffic=None) -> dict:
    peak, src = hbm_peak()
    ach = bytes_per_step / s_per_step / 1e9 if s_per_step > 0 else None
    out = {"bound": "hbm", "kernel": kernel, "achieved": ach, "peak": peak, "unit": "GB/s",
           "frac": ach / peak if ach else None, "algorithmic_bytes": bytes_per_step, "ms": 1e3 * s_per_step,
           "traffic": traffic, "peak_source": src}
    if note:
        out["note"] = note
    return out


def render_roofline(flops_per_view: float, views: int, k3_s: float, kernel: str, ktime=None) -> dict:
    """K3 against the FP32 pipe (8C + 6 (+8 with an aperture)
    flops per (view, bin, layer)).  achieved / frac: the step's flops over the
    main render tile's own launch durations (CUDA events recorded by the library
    around each launch, `fdl_kernel_timer`); *_stage: over the whole K3 stage
    k3_s (factor or z pre-pass + tile + Nyquist fix-up + launch gaps)."""
    ach_stage = flops_per_view * views / k3_s / 1e12 if k3_s > 0 else None
    out = {"bound": "fp32", "kernel": kernel, "achieved": ach_stage, "peak": FP32_PEAK_TFLOPS,
           "unit": "TFLOP/s", "frac": ach_stage / FP32_PEAK_TFLOPS if ach_stage else None,
           "flops_per_view": flops_per_view, "k3_ms": 1e3 * k3_s,
           "achieved_stage": ach_stage, "frac_stage": ach_stage / FP32_PEAK_TFLOPS if ach_stage else None,
           "peak_source": "measured FFMA2 (tools/microbench/fp32_pipes.cu); MEASURED_PEAKS.json has no fp32 entry"}
    if ktime and ktime["s_per_step"] > 0:
        ach = flops_per_view * views / ktime["s_per_step"] / 1e12
        out.update({"achieved": ach, "frac": ach / FP32_PEAK_TFLOPS, "kernel_ms_per_launch": ktime["ms_per_launch"],
                    "launches_per_step": ktime["launches_per_step"]})
    return out


def kernel_timer(on: bool):
    """Enable (clearing) / disable the library's per-launch events around K1 and K3."""
    from paper_1901_06919_b200 import _native as nat
    nat.lib().fdl_kernel_timer(1 if on else 0)


def kernel_time(which: int, steps: int):
    """{s_per_step, ms_per_launch, launches_per_step} of one timed kernel (0: K1, 1: K3), or None."""
    import ctypes
    from paper_1901_06919_b200 import _native as nat
    tot, cnt = ctypes.c_double(0.0), ctypes.c_int32(0)
    nat.check(nat.lib().fdl_kernel_timer_read(which, ctypes.byref(tot), ctypes.byref(cnt)), "fdl_kernel_timer_read")
    if cnt.value == 0:
        return None
    return {"s_per_step": tot.value / 1e3 / steps, "ms_per_launch": tot.value / cnt.value,
            "launches_per_step": cnt.value / steps}


def k1_traffic(cfg: str):
    try:
        return json.load(open(TRAFFIC_FILE)).get(cfg)
    except Exception:
        return None


def parallelism_note(world: int) -> str:
    return f"frequency-row slabs x{world} (chunked NCCL all-to-all), views x{world}" if world > 1 else "1 GPU"


L2_NOTE = "inputs (views, spectra, layers) exceed the 126 MB L2; no explicit flush"


def headline_config(m, H, W, C, n, pad, Q, c5_views, world) -> dict:
    """The `config` of the headline workload: identical in both arms (ours / --impl reference)."""
    return {"workload": f"c4+c5: c4: construct {m} views {H}x{W}x{C}, n={n} layers, pad {pad} (Q={Q} bins); then c5: "
                        f"render {c5_views} views of a 64-layer 1920x1080x3 FDL (disk(1), f=2r)",
            "bins": Q, "views": m, "layers": n, "channels": C, "render_views": c5_views,
            "parallelism": parallelism_note(world), "l2": L2_NOTE}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="headline")
    ap.add_argument("--size", type=int, default=None, help="override image size (testing)")
    ap.add_argument("--batch", type=int, default=64, help="render views per K3 launch (c1-c4 renders)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="also time the step as one CUDA-graph replay (paper_1901_06919_b200/graph.py); default on for c1")
    ap.add_argument("--cpu-sample-rows", type=int, default=None,
                    help="frequency rows solved per CPU sample step (default: 24, or 2 for c4)")
    ap.add_argument("--c5-views", type=int, default=C5_VIEWS, help="config 5: views rendered per step (all ranks)")
    ap.add_argument("--c5-batch", type=int, default=C5_BATCH, help="config 5: views per K3/K4 launch")
    ap.add_argument("--e2e-views", type=int, default=256, help="config 5: views per e2e render step")
    ap.add_argument("--sharded", action="store_true", help="use the multi-GPU code path even on one GPU")
    return ap.parse_args()


# ----------------------------------------------------------------------------- workloads
def canonical_flops_per_bin(cfg: str, m: int, n: int, C: int) -> float:
    """SURVEY.md §8(d) algorithmic fp64 flops per bin of K1."""
    if cfg == "c3":
        return 4 * m * n * C + m * n * (n + 1) + n ** 3 / 3 + 4 * n * n * C
    return 8 * m * n * C + 8 * m * n + (4.0 / 3.0) * n ** 3 + 8 * n * n * C


def make_workload(cfg, size, device):
    from harness.synth import make_case
    if cfg == "c3":
        from harness.focal import make_focal_case
        return make_focal_case(size, device=device)
    return make_case(cfg, size, device=device)


def synth_device():
    """Inputs are generated by the harness (torch, seeded) on the GPU when there
    is one, so both bench arms see the same data; only the generator runs there."""
    import torch
    return torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t0 = time.time()
            while time.time() - t0 < 3.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.remove(self.path)
        if not rows:
            return None
        sm = [r[0] for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in rows), "samples": len(rows),
                "reasons": reasons}


def merge_clocks(a, b):
    if not a or not b:
        return a or b
    n = a["samples"] + b["samples"]
    return {"sm_mhz": (a["sm_mhz"] * a["samples"] + b["sm_mhz"] * b["samples"]) / n,
            "sm_max_mhz": max(a["sm_max_mhz"], b["sm_max_mhz"]), "samples": n,
            "reasons": sorted(set(a["reasons"]) | set(b["reasons"])),
            "parts": {"construct": a, "render": b}}


def max_over_ranks(vals, device, world):
    if world == 1:
        return np.asarray(vals, dtype=np.float64)
    import torch
    import torch.distributed as dist
    t = torch.tensor(np.asarray(vals, dtype=np.float64), device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


# ----------------------------------------------------------------------------- C5 render sweep (ours)
def c5_model(size, device):
    import paper_1901_06919_b200 as fdl
    from harness.synth import random_fdl_layers
    H, W, n, C = (size or 1080), (int(size * 16 / 9) if size else 1920), 64, 3
    layers = random_fdl_layers(n, C, H, W, device=device)
    d = np.linspace(-5, 5, n)
    return fdl.FdlModel(disparities=d, layers=layers, grid=fdl.FrequencyGrid(W, H), width=W, height=H)


def c5_requests(count):
    import paper_1901_06919_b200 as fdl
    from harness.synth import render_requests_c5
    u, v, s, f = render_requests_c5(count)
    ap = fdl.aperture_spectrum("disk", diameter=1.0)
    return [fdl.RenderRequest(u=u[i], v=v[i], s=s[i], f=f[i], aperture=ap) for i in range(len(u))]


def run_c5(args, rank, world, device):
    """Config 5: render sweep over a precomputed random FDL (64 layers, 1920x1080 RGB):
    args.c5_views views per step split across the ranks, in args.c5_batch-view launches."""
    import importlib

    import torch
    import torch.distributed as dist

    R = importlib.import_module("paper_1901_06919_b200.render")
    model = c5_model(args.size, device)
    n, C, H = model.num_layers, model.layers_device().shape[1], model.height
    W = model.width
    reqs = c5_requests(args.c5_views)
    a, b = (len(reqs) * rank) // world, (len(reqs) * (rank + 1)) // world
    mine = reqs[a:b]
    batch = args.c5_batch
    stream = torch.cuda.current_stream()

    def step(timing=None):
        for b0 in range(0, len(mine), batch):
            R.render_many_device(model, mine[b0:b0 + batch], batch=batch, timing=timing)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(device.index or 0)
    sampler.start()
    torch.cuda.nvtx.range_push("timed")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rtim = []
    kernel_timer(True)
    e0.record(stream)
    for _ in range(args.steps):
        step(rtim)
    e1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    k3_kt = kernel_time(1, args.steps)
    kernel_timer(False)
    t_local = e0.elapsed_time(e1) / 1e3 / args.steps
    k3_s = sum(ev[0].elapsed_time(ev[1]) for ev in rtim) / 1e3 / args.steps
    k4_s = sum(ev[1].elapsed_time(ev[2]) for ev in rtim) / 1e3 / args.steps
    t, = max_over_ranks([t_local], device, world)
    Q = H * (W // 2 + 1)
    flops_view = Q * n * (8 * C + 6 + 8)
    V = len(mine)
    k4_bytes = V * (C * Q * 8 + H * W * C * 4)
    res = {"value": len(reqs) / t, "unit": "views/s", "ms": 1e3 * t, "views_per_step": len(reqs),
           "views_per_rank": V, "batch": batch,
           "stages_ms": {"k3_render_spectra_ms": 1e3 * k3_s, "k4_c2r_crop_ms": 1e3 * k4_s},
           "roofline": {**render_roofline(flops_view, V, k3_s, "K3 render tile (disk aperture, fp32 FFMA2)", k3_kt),
                        "traffic": k1_traffic("k3_c5") if batch == C5_BATCH else None},
           "k4_roofline": hbm_roofline("K4 inverse FFT + crop (mixed-radix engine: column pass + row pass)", k4_bytes,
                                       k4_s, "spectra read once (8 C Q B/view) + images written (4 H W C B/view); "
                                       "traffic: ncu DRAM bytes per 256-view launch",
                                       traffic=k1_traffic("k4_c5") if batch == C5_BATCH else None),
           "clocks": clocks,
           # per launch set: lookup pre-pass + TMA aperture tile + Nyquist-line fix-up + K4 column pass + K4 row pass
           "gpu_launches": args.steps * 5 * math.ceil(V / batch)}
    return res, model, reqs


def run_c5_e2e(args, model, reqs):
    """C5 through the public API: render_many -> float64 host images (the reference's
    output type), the model resident (a server that loaded it once)."""
    import torch
    import paper_1901_06919_b200 as fdl
    nv = min(args.e2e_views, len(reqs))
    steps = max(1, min(args.steps, 3))
    fdl.render_many(model, reqs[:nv], batch=64)  # warm (pinned host buffer, plans)
    torch.cuda.synchronize()
    ts = []
    for s in range(steps):
        sel = reqs[(s * nv) % len(reqs):(s * nv) % len(reqs) + nv]
        t0 = time.perf_counter()
        imgs = fdl.render_many(model, sel, batch=64)
        ts.append(time.perf_counter() - t0)
        del imgs
    H, W, C = model.height, model.width, model.layers_device().shape[1]
    return {"value": nv / float(np.mean(ts)), "unit": "views/s", "views_per_step": nv, "steps": steps,
            "h2d_bytes_per_step": nv * 4 * 8, "d2h_bytes_per_step": nv * H * W * C * 8,
            "note": "render_many, 64-view launches, float64 host images read back under the next batch's render"}


# ----------------------------------------------------------------------------- construction (ours)
def run_construct(args, cfg, rank, world, device, render=True):
    import torch
    import torch.distributed as dist

    import paper_1901_06919_b200 as fdl
    from paper_1901_06919_b200 import construct as K
    import importlib
    R = importlib.import_module("paper_1901_06919_b200.render")

    case = make_workload(cfg, args.size, device)
    views = case.views  # (m, H, W, C) float32 on the device
    m, H, W, C = views.shape
    d = case.d
    n = len(d)
    u, v = case.u, case.v
    wide = case.aperture is not None
    ap = fdl.aperture_spectrum(case.aperture["shape"], diameter=case.aperture["diameter"]) if wide else None
    vs_meta = fdl.ViewSet(images=np.zeros((m, 1, 1, C), np.float32), u=u, v=v, s=case.s,
                          apertures=[ap] * m if wide else None)
    pu, pv = np.outer(u, d), np.outer(v, d)
    pad = K.default_pad_margin(pu, pv)
    Hp, Wp = H + 2 * pad, W + 2 * pad
    Q = Hp * (Wp // 2 + 1)
    rc = case.render_coords if render else np.zeros((0, 2))
    reqs = [fdl.RenderRequest(u=float(a), v=float(b), f=0.0) for a, b in rc]
    V = len(reqs)
    stream = torch.cuda.current_stream()

    sharded = world > 1 or args.sharded
    if sharded:
        from paper_1901_06919_b200 import dist as D
        j0, j1 = D.view_range(m, world, rank)
        local_views = views[j0:j1].contiguous()
        shifts = fdl.ShiftParams.factored(u, v, d)
        my_reqs = reqs[(V * rank) // world:(V * (rank + 1)) // world]
        rows_local = D.slab_rows(Hp, world, rank)[0]
        Q_local = len(rows_local) * (Wp // 2 + 1)

    def construct_step(ev=None):
        """One construction; returns (slab layers or full layers, path)."""
        if sharded:
            layers_slab, rows, lam, _, _ = D.construct_sharded(local_views, j0, m, shifts, views_meta=vs_meta,
                                                               k1_events=ev)
            return layers_slab, 1
        spectra, sumsq = K.views_to_spectra(views, pad)
        if ev is not None:
            ev[2].record(stream)  # K0 done (pad + R2C + sum|b|^2)
            ev[0].record(stream)
        # default lambda on the device (construct_fdl does the same): no host round trip
        lam_dev = K.lambda_device(sumsq, Q, m)
        layers, nbad, path = K.solve_slab(spectra, m, n, C, Hp, Wp, np.arange(Hp), pu, pv, d, None, K.DEFAULT_EPS,
                                          views=vs_meta, u=None if wide else u, v=None if wide else v,
                                          lam_dev=lam_dev)
        if ev is not None:
            ev[1].record(stream)
        K.symmetrize(layers, Hp, Wp)
        return layers, path

    def to_model(layers):
        if sharded:  # replicate the layers for a view-sharded render (timed with the render)
            layers = D.gather_slabs(layers, Hp)
        return fdl.FdlModel(disparities=d, layers=layers, grid=fdl.FrequencyGrid(Wp, Hp), width=W, height=H,
                            pad_margin=pad)

    dev_batch = max(args.batch, V)  # device-resident renders: one launch set for the whole view set

    def render_step(layers, timing=None):
        model = to_model(layers)
        rq = my_reqs if sharded else reqs
        if rq:
            R.render_many_device(model, rq, batch=dev_batch, timing=timing)
        return model

    for _ in range(args.warmup):
        layers, path = construct_step()
        if V:
            render_step(layers)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(device.index if device.index is not None else 0)
    sampler.start()
    kernel_timer(True)
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ isolates the step's launches
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    rtim = []
    for s in range(args.steps):
        e = evs[s]
        e[0].record(stream)
        layers, path = construct_step(ev=(e[3], e[4], e[5]))
        e[1].record(stream)
        if V:
            render_step(layers, timing=rtim)
        e[2].record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    k1_kt, k3_kt = kernel_time(0, args.steps), kernel_time(1, args.steps)
    kernel_timer(False)
    t_con = np.array([e[0].elapsed_time(e[1]) for e in evs]) / 1e3
    t_ren = np.array([e[1].elapsed_time(e[2]) for e in evs]) / 1e3
    t_k1 = np.array([e[3].elapsed_time(e[4]) for e in evs]) / 1e3
    stages = {}
    if not sharded:
        stages["k0_pack_fft_sumsq_ms"] = float(np.mean([e[0].elapsed_time(e[5]) for e in evs]))
        stages["k1_ms"] = float(np.mean(t_k1)) * 1e3
        stages["k2_symmetrize_ms"] = float(np.mean([e[4].elapsed_time(e[1]) for e in evs]))
    if rtim:
        stages["k3_render_spectra_ms"] = float(sum(t[0].elapsed_time(t[1]) for t in rtim)) / args.steps
        stages["k4_c2r_crop_ms"] = float(sum(t[1].elapsed_time(t[2]) for t in rtim)) / args.steps
    t_con_mean, t_ren_mean, t_k1_mean = max_over_ranks([t_con.sum(), t_ren.sum(), t_k1.sum()], device,
                                                       world) / args.steps

    assert torch.isfinite(torch.view_as_real(layers)).all().item(), "non-finite layers"

    F_bin = canonical_flops_per_bin(cfg, m, n, C)
    q_k1 = Q_local if sharded else Q  # bins one K1 launch solves on this rank
    achieved_stage = F_bin * q_k1 / t_k1_mean / 1e12  # over the K1 stage (tables, solve, status count)
    achieved = F_bin * q_k1 / k1_kt["s_per_step"] / 1e12 if k1_kt else achieved_stage  # solve kernel launches
    value = Q * n / t_con_mean  # the whole job's bins per max-over-ranks time
    whp = Wp // 2 + 1
    res = {
        "metric": METRIC,
        "value": value,
        "unit": "freq·layers/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * (t_con_mean + t_ren_mean),
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f64 solve / c64 I/O / f32 render",
        "data": "synthetic (harness/synth.py seeded occluded layered scene, SURVEY.md §8(d))",
        "config": {"workload": f"{cfg}: construct {m} views {H}x{W}x{C}, n={n} layers, pad {pad} "
                               f"(Q={Q} bins)" + (f", then render {V} views" if V else ""),
                   "bins": Q, "views": m, "layers": n, "channels": C, "render_views": V,
                   "parallelism": parallelism_note(world), "l2": L2_NOTE},
        "k1_path": int(path),
        "construct_ms": 1e3 * t_con_mean,
        "stages_ms": stages,
        "k1_ms": 1e3 * t_k1_mean,
        "roofline": {"bound": "tensor", "kernel": "k1_fast_kernel (fp64 DMMA)",
                     "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS,
                     "kernel_ms_per_launch": k1_kt["ms_per_launch"] if k1_kt else None,
                     "launches_per_step": k1_kt["launches_per_step"] if k1_kt else None,
                     "achieved_stage": achieved_stage, "frac_stage": achieved_stage / FP64_PEAK_TFLOPS,
                     "traffic": k1_traffic(cfg) if world == 1 else None,
                     "algorithmic_bytes": 8 * C * (m + n) * q_k1,
                     "flops_per_bin": F_bin,
                     # `achieved` counts the CANONICAL flops of the reference's complex solve;
                     # the real re-writes execute roughly a quarter of them, so frac can exceed 1 while the
                     # fp64 pipe is far from busy (ncu sm__pipe_fp64_cycles_active on C4, same kernel)
                     "frac_counts": "canonical flops (the executed count is lower; see pipe_active_ncu)",
                     "pipe_active_ncu": k1_traffic("k1_c4_fp64_pipe_active_ncu") if cfg in ("c4", "headline") else None,
                     "peak_source": "measured fp64 DMMA m8n8k4 (profiles/r01_fp64_pipes.txt); "
                                    "MEASURED_PEAKS.json has no fp64 entry"},
        "clocks": clocks,
        # K0 (rows + cols + per-view sums) 3, default lambda 1, K1 (axis tables + solve + residual screen +
        # status count) 4, K2 1; renders: z tables + tile + Nyquist fix-up + K4 column pass + K4 row pass = 5
        # per launch set
        "gpu_launches": args.steps * ((9 + world if sharded else 9)
                                      + 5 * math.ceil((V // world + 1 if sharded else V) / dev_batch)),
    }
    if not sharded:
        k0_s = stages["k0_pack_fft_sumsq_ms"] / 1e3
        res["k0_roofline"] = hbm_roofline("K0 pad + R2C + sum|b|^2 (FFT engine rows + columns)",
                                          m * H * W * C * 4 + m * C * Q * 8, k0_s,
                                          "views read once (4 m H W C B) + spectra written once (8 m C Q B); "
                                          "traffic: ncu DRAM bytes per construction (row pass + column pass)",
                                          traffic=k1_traffic("k0_" + cfg))
    if V:
        res["render"] = {"value": V / t_ren_mean, "unit": "views/s", "ms": 1e3 * t_ren_mean,
                         "roofline": render_roofline(Q * n * (8 * C + 6), V // world if world > 1 else V,
                                                     stages.get("k3_render_spectra_ms", 0.0) / 1e3,
                                                     "K3 render tile (pinhole, fp32 FFMA2)", k3_kt)}
        if "k4_c2r_crop_ms" in stages:
            res["render"]["k4_roofline"] = hbm_roofline(
                "K4 inverse FFT + crop", V * (C * Q * 8 + H * W * C * 4), stages["k4_c2r_crop_ms"] / 1e3,
                "spectra read once + images written once")
    if (args.graph or cfg == "c1") and not sharded and not wide:
        res["graph"] = run_graphed(args, case, reqs, Q, n)
    return res, case, (m, n, C, H, W, pad, Hp, Wp, Q, V)


def run_graphed(args, case, reqs, Q, n):
    """The same step (construction + renders) as ONE CUDA-graph replay for a fixed geometry."""
    import importlib
    import torch
    import paper_1901_06919_b200 as fdl
    G = importlib.import_module("paper_1901_06919_b200.graph")
    views = fdl.ViewSet(images=case.views, u=case.u, v=case.v)
    g = G.GraphedConstruct(views, fdl.ShiftParams.factored(case.u, case.v, case.d), requests=reqs)
    for _ in range(max(args.warmup, 3)):
        g()
    g.check()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        g()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    return {"ms_per_step": ms, "value": Q * n / (ms / 1e3), "unit": "freq·layers per second of whole step",
            "note": "construction + renders of the step as one CUDA-graph replay (views already in HBM; the host-driven "
                    "fallbacks are replaced by a status check, GraphedConstruct.check)"}


def run_construct_e2e(args, case, dims, device, host_views=None):
    """Same construction (and renders) through the public API from pinned host buffers."""
    import torch

    import paper_1901_06919_b200 as fdl
    m, n, C, H, W, pad, Hp, Wp, Q, V = dims
    if host_views is None:
        host_views = torch.empty(tuple(case.views.shape), dtype=torch.float32, pin_memory=True)
        host_views.copy_(case.views.cpu())
    wide = case.aperture is not None
    ap = fdl.aperture_spectrum(case.aperture["shape"], diameter=case.aperture["diameter"]) if wide else None
    vs = fdl.ViewSet(images=host_views, u=case.u, v=case.v, s=case.s, apertures=[ap] * m if wide else None)
    sh = fdl.ShiftParams.factored(case.u, case.v, case.d)
    reqs = [fdl.RenderRequest(u=float(a), v=float(b), f=0.0) for a, b in case.render_coords] if V else []

    def step():
        t0 = time.perf_counter()
        model = fdl.construct_fdl(vs, sh)
        res = model.layers_host()  # the layers in host memory (read back slab by slab during the solve)
        assert tuple(res.shape) == (n, C, Hp, Wp // 2 + 1)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if reqs:
            fdl.render_many(model, reqs, batch=args.batch)
        t2 = time.perf_counter()
        del model, res
        return t1 - t0, t2 - t1

    big = m * H * W * C * 4 > (4 << 30)
    steps = max(1, min(args.steps, 5)) if big else args.steps
    for _ in range(1 if big else max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    tc, tr = [], []
    for _ in range(steps):
        a, b = step()
        tc.append(a)
        tr.append(b)
    out = {"value": Q * n / float(np.mean(tc)), "unit": "freq·layers/s", "steps": steps,
           "h2d_bytes_per_step": int(host_views.numel() * 4),
           "d2h_bytes_per_step": int(n * C * Q * 8) + V * H * W * C * 8,
           "construct_ms": 1e3 * float(np.mean(tc))}
    if V:
        out["render"] = {"value": V / float(np.mean(tr)), "unit": "views/s", "ms": 1e3 * float(np.mean(tr)),
                         "d2h_bytes_per_step": V * H * W * C * 8}  # float64 images, like the reference
    if big and not wide:
        # the same construction from 8-bit host views (the loader's on-disk format, reference io.py:54-59),
        # decoded on the device: a secondary figure, the headline e2e stays on float32 host views
        q8 = torch.empty(tuple(host_views.shape), dtype=torch.uint8, pin_memory=True)
        for j in range(m):
            q8[j].copy_((host_views[j].clamp(0, 1) * 255).round().to(torch.uint8))
        vq = fdl.ViewSet(images=fdl.QuantisedImages(q8), u=case.u, v=case.v, s=case.s)

        def qstep():
            t0 = time.perf_counter()
            model = fdl.construct_fdl(vq, sh)
            res = model.layers_host()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            del model, res
            return dt

        qstep()
        tq = [qstep() for _ in range(steps)]
        out["quantised_views"] = {"value": Q * n / float(np.mean(tq)), "unit": "freq·layers/s",
                                  "construct_ms": 1e3 * float(np.mean(tq)), "h2d_bytes_per_step": int(q8.numel()),
                                  "note": "uint8 host views (QuantisedImages), decoded by fdl_dequantise_views"}
        del q8, vq
    return out


# ----------------------------------------------------------------------------- CPU (oracle) samples
def _cores(c0, w0):
    return round((time.process_time() - c0) / max(time.perf_counter() - w0, 1e-9), 2)


def spectra_rows_partial_dft(host_views, pad, rows, Hp, Wp):
    """Spectrum rows `rows` of every padded view, (len(rows), Whp, m, C) complex128,
    by a partial DFT (column sums against exp(-2 pi i r y / Hp), then an rfft along x):
    the same values as rows of rfft2 of the padded views (construct.py:253-263) to
    rounding, without transforming whole views.  Untimed input preparation of the
    C4 slab sample."""
    hv = np.asarray(host_views)
    m, H, W, C = hv.shape
    y = np.arange(H) + pad
    E = np.exp(-2j * np.pi * np.outer(np.asarray(rows, float), y) / Hp)  # (R, H)
    Er, Ei = np.ascontiguousarray(E.real), np.ascontiguousarray(E.imag)
    whp = Wp // 2 + 1
    out = np.empty((len(rows), whp, m, C), dtype=np.complex128)
    for j in range(m):
        img = hv[j].reshape(H, W * C).astype(np.float64)
        z = (Er @ img + 1j * (Ei @ img)).reshape(len(rows), W, C)
        zp = np.zeros((len(rows), Wp, C), dtype=np.complex128)
        zp[:, pad:pad + W] = z
        out[:, :, j, :] = np.fft.fft(zp, axis=1)[:, :whp]
    return out


class C4Sample:
    """Bounded sample of the reference construction on the host (SURVEY.md §8(c) slab
    oracle): per step, the rfft2 (+ sum|b|^2) of one padded view and the per-bin
    solves of one mirrored frequency-row pair, extrapolated to all m views and all
    Q bins (per-bin results are chunk-independent, test_construct.py:196-204)."""

    def __init__(self, host_views, case, dims, rows_per_step=2):
        from oracle import fdl_oracle as O
        self.O = O
        m, n, C, H, W, pad, Hp, Wp, Q, V = dims
        self.dims = dims
        self.hv = host_views
        self.pu, self.pv = np.outer(case.u, case.d), np.outer(case.v, case.d)
        self.d = case.d
        half = max(1, rows_per_step // 2)
        self.rows = np.array(sorted(set([r for k in range(1, half + 1) for r in (k, Hp - k)])))
        self.b_rows = spectra_rows_partial_dft(host_views, pad, self.rows, Hp, Wp)
        # lambda of the full problem (any positive value gives the same solve cost);
        # from the sampled rows' energy, scaled to the whole grid
        self.lam = O.default_lam(np.sum(np.abs(self.b_rows.reshape(-1, m, C)) ** 2, axis=(1, 2)), m)
        self.i = 0

    def step(self):
        O = self.O
        m, n, C, H, W, pad, Hp, Wp, Q, V = self.dims
        j = self.i % m
        self.i += 1
        t0 = time.perf_counter()
        b, _, _ = O.view_spectra(np.asarray(self.hv[j:j + 1]), pad)
        float(np.sum(np.abs(b) ** 2))
        t1 = time.perf_counter()
        O.solve_rows(self.b_rows, self.rows, self.pu, self.pv, self.d, self.lam, Hp, Wp)
        t2 = time.perf_counter()
        nb = len(self.rows) * (Wp // 2 + 1)
        return (t1 - t0) * m + (t2 - t1) * Q / nb

    def describe(self):
        m, n, C, H, W, pad, Hp, Wp, Q, V = self.dims
        nb = len(self.rows) * (Wp // 2 + 1)
        return (f"per step: rfft2 + sum|b|^2 of 1 of {m} padded views (x{m}) and the solves of {len(self.rows)} "
                f"mirrored frequency rows = {nb} of {Q} bins (x{Q / nb:.0f}); row spectra by a partial DFT "
                "(untimed)")


class C5Sample:
    """Bounded sample of the reference render on the host: one C5 request per step
    (render.py:228-248 restated: aperture lookups, weighted layer sum, irfft2, crop)."""

    def __init__(self, model, reqs):
        from oracle import fdl_oracle as O
        self.O = O
        self.layers = model.layers_host().numpy().astype(np.complex128)
        self.d = np.asarray(model.disparities, float)
        self.H, self.W = model.height, model.width
        self.tab = O.aperture_table("disk", diameter=1.0)
        self.reqs = reqs
        self.i = 0

    def step(self):
        r = self.reqs[self.i % len(self.reqs)]
        self.i += 1
        t0 = time.perf_counter()
        self.O.render(self.layers, self.d, self.H, self.W, 0, self.H, self.W, u=r.u, v=r.v, s=r.s, f=r.f,
                      ap=self.tab)
        return time.perf_counter() - t0


def cpu_baseline_headline(c4s, c5s, steps=1):
    c0, w0 = time.process_time(), time.perf_counter()
    t4 = float(np.mean([c4s.step() for _ in range(steps)]))
    cores4 = _cores(c0, w0)
    c0, w0 = time.process_time(), time.perf_counter()
    t5 = float(np.mean([c5s.step() for _ in range(steps)])) if c5s is not None else None
    cores5 = _cores(c0, w0)
    m, n, C, H, W, pad, Hp, Wp, Q, V = c4s.dims
    return {"value": Q * n / t4, "unit": "freq·layers/s", "cores": max(cores4, cores5), "kind": "port",
            "sample": c4s.describe() + (f"; render: 1 C5 request per step" if c5s is not None else ""),
            "construct_s_extrapolated": t4,
            "render_views_per_s": (1.0 / t5) if t5 else None, "cores_construct": cores4, "cores_render": cores5}


def cpu_sample(args, case, dims, n_steps=1):
    """c1-c3: the reference algorithm on the host: full view FFTs + lambda, the per-bin
    solves of a bounded sample of mirrored frequency-row pairs, extrapolated by bin count;
    plus a few renders."""
    from oracle import fdl_oracle as O
    m, n, C, H, W, pad, Hp, Wp, Q, V = dims
    views = case.views.cpu().numpy().astype(np.float64)
    pu, pv = np.outer(case.u, case.d), np.outer(case.v, case.d)
    views_ap = None
    if case.aperture is not None:
        tab = O.aperture_table(case.aperture["shape"], diameter=case.aperture["diameter"])
        views_ap = [(tab, float(case.s[j]), 1.0) for j in range(m)]
    whp = Wp // 2 + 1
    nrow = max(2, min(args.cpu_sample_rows or 24, Hp))
    rows = np.unique(np.concatenate([np.arange(1, nrow // 2 + 1), Hp - np.arange(1, nrow // 2 + 1)]))
    t_con, t_ren = [], []
    c0 = time.process_time()
    w0 = time.perf_counter()
    for _ in range(n_steps):
        t0 = time.perf_counter()
        b_all, hp, wp = O.view_spectra(views, pad)
        lam = O.default_lam(np.sum(np.abs(b_all) ** 2, axis=(1, 2)), m)
        t1 = time.perf_counter()
        b_rows = b_all.reshape(Hp, whp, m, C)[rows]
        O.solve_rows(b_rows, rows, pu, pv, case.d, lam, Hp, Wp, views_ap=views_ap)
        t2 = time.perf_counter()
        t_con.append((t1 - t0) + (t2 - t1) * Hp / len(rows))
        layers = np.zeros((n, C, Hp, whp), dtype=np.complex128)
        r0 = time.perf_counter()
        nr = 2
        for (a, b) in case.render_coords[:nr]:
            O.render(layers, case.d, Hp, Wp, pad, H, W, u=a, v=b)
        t_ren.append((time.perf_counter() - r0) / nr)
    cores = _cores(c0, w0)
    sample = (f"full view FFTs + lambda, per-bin solves of {len(rows)} of {Hp} frequency rows "
              f"(extrapolated x{Hp / len(rows):.1f}), {2} renders per step")
    return float(np.mean(t_con)), float(np.mean(t_ren)), cores, sample


def c4_dims(case):
    m, H, W, C = case.views.shape
    n = len(case.d)
    pu, pv = np.outer(case.u, case.d), np.outer(case.v, case.d)
    pad = int(math.ceil(max(np.abs(pu).max(), np.abs(pv).max())))
    Hp, Wp = H + 2 * pad, W + 2 * pad
    return (m, n, C, H, W, pad, Hp, Wp, Hp * (Wp // 2 + 1), 0)


def host_copy(t):
    import torch
    h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h


# ----------------------------------------------------------------------------- headline (ours)
def run_headline(args, rank, world, device):
    import torch
    res, case, dims = run_construct(args, "c4", rank, world, device, render=False)
    m_, n_, C_, H_, W_, pad_ = dims[:6]  # dims = (m, n, C, H, W, pad, Hp, Wp, Q, V)
    res["config"] = headline_config(m_, H_, W_, C_, n_, pad_, dims[8], args.c5_views, world)
    res["render_batch"] = args.c5_batch
    host_views = None
    c4s = None
    if world == 1:
        host_views = host_copy(case.views)
        if not args.no_e2e:
            res["e2e"] = run_construct_e2e(args, case, dims, device, host_views=host_views)
        torch.cuda.empty_cache()
        if rank == 0 and not args.no_cpu_baseline:
            c4s = C4Sample(host_views, case, dims, rows_per_step=args.cpu_sample_rows or 2)
    del case
    torch.cuda.empty_cache()
    r5, model5, reqs5 = run_c5(args, rank, world, device)
    clocks4 = res.get("clocks")
    res["clocks"] = merge_clocks(clocks4, r5.pop("clocks"))
    res["gpu_launches"] += r5.pop("gpu_launches")
    res["render"] = r5
    res["ms_per_step"] = res["construct_ms"] + r5["ms"]
    if world == 1 and not args.no_e2e:
        res["e2e"]["render"] = run_c5_e2e(args, model5, reqs5)
    if c4s is not None:
        c5s = C5Sample(model5, reqs5)
        res["cpu_baseline"] = cpu_baseline_headline(c4s, c5s, steps=1)
    return res


# ----------------------------------------------------------------------------- calibration
def calib_flops_per_bin(m: int, n: int, grad: bool) -> float:
    """fp64 flops of one calibration bin evaluation (calibrate.py:139-229): Hermitian
    Gram 4mn(n+1), RHS 8mn, Cholesky (4/3)n^3, two solves 8n^2, residual 8mn,
    Gamma x 2n^2 (+ gradient 8mn); the phase generation is not counted."""
    return 4 * m * n * (n + 1) + 8 * m * n + (4.0 / 3.0) * n ** 3 + 8 * n * n + 8 * m * n + 2 * n * n + (
        8 * m * n if grad else 0)


CALIB_BATCH = 4096  # CalibConfig.batch_size default (calibrate.py:65)


def calib_case(args, device):
    """Calibration workload: the config-2 light field (81 views 512x512 RGB), 30 layers,
    one descent iteration = the gradient evaluation + one backtracking trial over a
    4096-bin batch of the frequency pool (calibrate.py:378-392)."""
    from harness.synth import make_case
    case = make_case("c2", args.size, device=device)
    rng = np.random.default_rng(7)
    m, n = len(case.u), len(case.d)
    u = case.u + 0.02 * rng.standard_normal(m)
    v = case.v + 0.02 * rng.standard_normal(m)
    return case, np.outer(u, case.d), np.outer(v, case.d), rng


def run_calib(args, device):
    """--config calib: GPU calibration iterations (paper_1901_06919_b200.calibrate, K5)."""
    import torch
    import paper_1901_06919_b200 as fdl
    import importlib
    CAL = importlib.import_module("paper_1901_06919_b200.calibrate")
    case, pu, pv, rng = calib_case(args, device)
    m, H, W, C = case.views.shape
    n = pu.shape[1]
    views = fdl.ViewSet(images=case.views.cpu().numpy(), u=case.u, v=case.v)
    spectra = CAL._Spectra(views)
    pool = CAL.frequency_pool(spectra.grid)
    spectra.normalise(pool)
    eng = CAL._Engine(spectra, n, CAL.layer_regularizer(n), CAL.DEFAULT_LAMBDA)
    batches = [np.sort(rng.permutation(pool)[:CALIB_BATCH]) for _ in range(4)]
    trial_pu, trial_pv = pu * 1.001, pv * 1.001

    def step(i):
        sel = batches[i % len(batches)]
        eng.batch_objective(pu, pv, sel, grad=True)
        eng.batch_objective(trial_pu, trial_pv, sel)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    sampler = ClockSampler(device.index or 0)
    sampler.start()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    t = e0.elapsed_time(e1) / 1e3 / args.steps
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sel = batches[0]
    k0.record(stream)
    eng.solve(pu, pv, sel)
    k1.record(stream)
    torch.cuda.synchronize()
    ts = k0.elapsed_time(k1) / 1e3
    flops = CALIB_BATCH * (calib_flops_per_bin(m, n, True) + calib_flops_per_bin(m, n, False))
    dfma_peak = 34.2
    res = {"metric": "calibration descent: frequency-bin evaluations/s (config-2 views)",
           "value": 2 * CALIB_BATCH / t, "unit": "bin-evaluations/s", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (harness/synth.py config-2 light field, perturbed grid coordinates)",
           "config": {"workload": f"calib: {m} views {H}x{W}x{C} (luminance), n={n} layers, one descent iteration = "
                                  f"gradient + one trial evaluation of a {CALIB_BATCH}-bin batch",
                      "batch": CALIB_BATCH, "l2": "spectra (Q x m complex128, 170 MB) exceed L2"},
           "solve_ms": 1e3 * ts,
           "roofline": {"bound": "fp64", "kernel": "K5 calibration solve + terms (DFMA)",
                        "achieved": flops / t / 1e12, "peak": dfma_peak, "unit": "TFLOP/s",
                        "frac": flops / t / 1e12 / dfma_peak,
                        "peak_source": "measured DFMA (tools/microbench/fp64_pipes.cu)",
                        "note": "step time includes the host descent bookkeeping and one device->host read per evaluation"},
           "clocks": clocks, "gpu_launches": args.steps * 2 * 4,
           "e2e": {"value": 2 * CALIB_BATCH / t, "unit": "bin-evaluations/s",
                   "h2d_bytes_per_step": 2 * (CALIB_BATCH * 4 + 2 * m * n * 8),
                   "d2h_bytes_per_step": 2 * 8 + 2 * m * n * 8}}
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = calib_cpu(args, case, pu, pv, batches[0])
    return res


def calib_cpu(args, case, pu, pv, sel, steps=1):
    """The reference's batch evaluation (oracle restatement of calibrate.py:139-229) on the host."""
    from oracle import fdl_oracle as O
    imgs = case.views.cpu().numpy().astype(np.float64)
    m, H, W, C = imgs.shape
    n = pu.shape[1]
    spec = O.luma_spectra(imgs)
    gamma = O.layer_regularizer(n)
    sample = sel[:512]
    c0, w0 = time.process_time(), time.perf_counter()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.calib_batch(pu, pv, spec, sample, W, H, 1e-3, gamma, grad=True)
        O.calib_batch(pu * 1.001, pv * 1.001, spec, sample, W, H, 1e-3, gamma)
        ts.append(time.perf_counter() - t0)
    return {"value": 2 * len(sample) / float(np.mean(ts)), "unit": "bin-evaluations/s", "cores": _cores(c0, w0),
            "kind": "port", "sample": f"gradient + trial evaluation of {len(sample)} of the batch's bins"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """--impl reference: the reference CPU algorithm (oracle port) on the host cores,
    same config, metric and seeded inputs as our arm; rank 0 only."""
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    if args.config == "calib":
        case, pu, pv, rng = calib_case(args, "cpu")
        sel = np.sort(rng.permutation(np.arange(case.views.shape[1] * (case.views.shape[2] // 2 + 1)))[:CALIB_BATCH])
        cb = calib_cpu(args, case, pu, pv, sel, steps=max(1, args.steps))
        return {"impl": "reference", "metric": "calibration descent: frequency-bin evaluations/s (config-2 views)",
                "value": cb["value"], "unit": cb["unit"], "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * 2 * 512 / cb["value"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "calib (oracle port of calibrate.py:139-229)", "batch": 512},
                "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if args.config == "headline":
        return run_reference_headline(args)
    dev = synth_device()
    case = make_workload(args.config, args.size, dev)
    case.views = case.views.cpu()
    m, H, W, C = case.views.shape
    n = len(case.d)
    pu, pv = np.outer(case.u, case.d), np.outer(case.v, case.d)
    pad = int(math.ceil(max(np.abs(pu).max(), np.abs(pv).max())))
    Hp, Wp = H + 2 * pad, W + 2 * pad
    Q = Hp * (Wp // 2 + 1)
    V = len(case.render_coords)
    dims = (m, n, C, H, W, pad, Hp, Wp, Q, V)
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    for _ in range(args.warmup and 1):
        cpu_sample(args, case, dims)
    t_con, t_ren, cores, sample = cpu_sample(args, case, dims, n_steps=args.steps)
    value = Q * n / t_con
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": value, "unit": "freq·layers/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * (t_con + V * t_ren), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: construct {m} views {H}x{W}x{C}, n={n} layers, pad {pad} "
                               f"(Q={Q} bins), then render {V} views", "bins": Q, "render_views": V},
        "render": {"value": 1.0 / t_ren, "unit": "views/s"},
        "cpu_baseline": {"value": value, "unit": "freq·layers/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "freq·layers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_reference_headline(args):
    """C4 construction + C5 render of the reference algorithm on bounded samples (C4Sample,
    C5Sample), the inputs generated by the same seeded harness as our arm."""
    import torch
    dev = synth_device()
    case = make_workload("c4", args.size, dev)
    dims = c4_dims(case)
    m, n, C, H, W, pad, Hp, Wp, Q, V = dims
    host_views = case.views.cpu().numpy()
    del case.views
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    c4s = C4Sample(host_views, case, dims, rows_per_step=args.cpu_sample_rows or 2)
    model5 = c5_model(args.size, dev)
    reqs5 = c5_requests(args.c5_views)
    c5s = C5Sample(model5, reqs5)
    del model5
    for _ in range(min(args.warmup, 1)):
        c4s.step()
        c5s.step()
    c0, w0 = time.process_time(), time.perf_counter()
    t4 = float(np.mean([c4s.step() for _ in range(args.steps)]))
    cores4 = _cores(c0, w0)
    c0, w1 = time.process_time(), time.perf_counter()
    t5 = float(np.mean([c5s.step() for _ in range(args.steps)]))
    cores5 = _cores(c0, w1)
    wall_ms = 1e3 * (time.perf_counter() - w0) / max(1, args.steps)  # what one sampled step really took
    value = Q * n / t4
    sample = c4s.describe() + "; render: 1 C5 request per step"
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "freq·layers/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall_ms,
        "full_step_ms_extrapolated": 1e3 * (t4 + args.c5_views * t5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (harness/synth.py seeded occluded layered scene, SURVEY.md §8(d)); same seeds and "
                "generator device as our arm",
        "config": headline_config(m, H, W, C, n, pad, Q, args.c5_views, args.gpus),
        "render": {"value": 1.0 / t5, "unit": "views/s", "s_per_view": t5},
        "construct_s_extrapolated": t4,
        "cpu_baseline": {"value": value, "unit": "freq·layers/s", "cores": max(cores4, cores5), "kind": "port",
                         "sample": sample, "render_views_per_s": 1.0 / t5},
        "e2e": {"value": value, "unit": "freq·layers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ----------------------------------------------------------------------------- main
def main():
    args = parse()
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            print(json.dumps(res))
        return
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        print(json.dumps({"error": "no CUDA device"}))
        sys.exit(1)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1 or args.sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=device)
    if args.config == "calib":
        if rank == 0:
            print(json.dumps(run_calib(args, device)))
        return
    if args.config == "headline":
        res = run_headline(args, rank, world, device)
    elif args.config == "c5":
        r5, model, reqs = run_c5(args, rank, world, device)
        res = {"metric": "rendered views/s (config 5)", "value": r5["value"], "unit": "views/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": r5["ms"], "higher_is_better": True,
               "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32 render",
               "data": "synthetic random FDL (harness/synth.py random_fdl_layers, render_requests_c5)",
               "config": {"workload": f"c5: render {args.c5_views} views of a 64-layer FDL, disk(1) f=2r",
                          "views_per_step": args.c5_views},
               **{k: r5[k] for k in ("stages_ms", "roofline", "k4_roofline", "clocks", "gpu_launches")}}
        if world == 1 and not args.no_e2e:
            res["e2e"] = run_c5_e2e(args, model, reqs)
    else:
        res, case, dims = run_construct(args, args.config, rank, world, device)
        if not args.no_e2e and world == 1:
            res["e2e"] = run_construct_e2e(args, case, dims, device)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            t_con, t_ren, cores, sample = cpu_sample(args, case, dims)
            res["cpu_baseline"] = {"value": dims[8] * dims[1] / t_con, "unit": "freq·layers/s", "cores": cores,
                                   "kind": "port", "sample": sample, "render_views_per_s": 1.0 / t_ren}
    if rank == 0:
        print(json.dumps(res))
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

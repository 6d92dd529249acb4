"""bench.py — measures the generalized sparse convolution hot path (arXiv 1904.08755) on B200.

One step = one pass of every §8(a) row of SURVEY.md over one ScanNet-shaped scan
(BASELINE.json configs[1]): quantize ~1M float points at 2 cm into a coordinate hash table
(a1, a2), build the 3x3x3 kernel map (a4, a5), then conv forward, input gradient and weight
gradient at C = 64 -> 64 in bf16 on the tcgen05 tensor cores (a6-a8).  Inputs are resident
in HBM when the timed region starts; L2 is flushed (256 MiB write, untimed) before every
timed step; each step is timed with CUDA events on the launching stream.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mk|reference]
Under torchrun (N > 1) every rank runs its own scan (weak scaling, batch-index sharding,
SURVEY §8(e)); the only collective is the NCCL all-reduce of dW (data-parallel gradient sum).
`--impl reference` times the CPU oracle (oracle/, the only other place bench.py runs it).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]
UNIT = "TFLOP/s"
C_IN = C_OUT = 64
K_OFF = 27


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mk", choices=["mk", "reference"])
    ap.add_argument("--seed", type=int, default=2000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.time(), parts))

    def stop(self, t0, t1):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        rows = [r for (t, r) in self.rows if t0 - 0.06 <= t <= t1 + 0.06] or [r for (_, r) in self.rows[-3:]]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def step_config(N, M, n_points, seed, ws):
    """The `config` of the bench line (shared by the GPU arm and the --impl reference arm)."""
    return {"workload": "configs[1]: ScanNet-shaped room, 2 cm voxels, 3x3x3 hypercube, C 64->64, "
                        "quantize + hash + kernel map + fwd + dgrad + wgrad",
            "voxels_per_gpu": int(N), "pairs_per_gpu": int(M), "points_per_gpu": int(n_points),
            "seed": seed, "parallelism": f"batch-index dp{ws}",
            "l2": "flushed before every timed step (256 MiB write, outside the step events)"}


def workload(seed):
    import synthetic
    pts = synthetic.room_points(seed)
    return pts


# ---------------------------------------------------------------------------- GPU arm
def run_mk(args, ws, rank, local):
    import torch
    import torch.distributed as dist

    import paper_1904_08755_b200 as mk
    import synthetic
    from paper_1904_08755_b200.dist import allreduce_grad

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    region = mk.Region(mk.HYPERCUBE, 3, 3)

    # ---- synthetic inputs (each rank its own scan: weak scaling by batch-index sharding)
    pts_h = workload(args.seed + rank)
    pts = torch.from_numpy(pts_h).to(dev)
    c0, _, _ = mk.coords_quantize(pts, synthetic.ROOM_VOXEL)
    N = c0.n
    m0 = mk.kmap_build(c0, c0, region)
    M = m0.n_pairs
    del m0, c0
    X = torch.from_numpy(synthetic.features(1, N, C_IN)).to(dev).to(torch.bfloat16)
    W = torch.from_numpy(synthetic.weights(2, K_OFF, C_OUT, C_IN)).to(dev).to(torch.bfloat16)
    G = torch.from_numpy(synthetic.features(3, N, C_OUT)).to(dev).to(torch.bfloat16)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    flops_pass = 2.0 * C_IN * C_OUT * M  # one of fwd / dgrad / wgrad
    flops_step = 3.0 * flops_pass

    def step(ev=None):
        def mark(i):
            if ev is not None:
                ev[i].record(stream)
        mark(0)
        # a1, a2 (deferred row count: the map build collects it, the host runs ahead meanwhile)
        c, _, _ = mk.coords_quantize(pts, synthetic.ROOM_VOXEL, return_maps=True, deferred=True)
        mark(1)
        m = mk.kmap_build(c, c, region)                                             # a4, a5
        mark(2)
        y = mk.conv_forward(m, X, W)                                                # a6
        mark(3)
        gin, _ = mk.conv_backward(m, G, X, W, need_gin=True, need_gw=False)          # a7
        mark(4)
        _, gw = mk.conv_backward(m, G, X, W, need_gin=False, need_gw=True)           # a8
        mark(5)
        if ws > 1:
            allreduce_grad(gw)  # data-parallel weight-gradient sum over NVLink (NCCL)
        mark(6)
        return y, gin, gw

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    n_ev = 7
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)] for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    launches0 = mk.kernel_launch_count()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    for i in range(args.steps):
        flush.zero_()  # L2 flush (untimed: outside the step's events)
        step(evs[i])
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t1 = time.time()
    launches = mk.kernel_launch_count() - launches0
    clocks = sampler.stop(t0, t1)

    ph = np.array([[evs[i][j].elapsed_time(evs[i][j + 1]) for j in range(n_ev - 1)] for i in range(args.steps)])
    step_ms = ph.sum(axis=1)
    total_ms = float(step_ms.sum())
    if ws > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = ws * flops_step / (ms_per_step * 1e-3) / 1e12
    mean_ph = ph.mean(axis=0)
    names = ["quantize", "kmap", "conv_fwd", "conv_dgrad", "conv_wgrad", "allreduce_dW"]
    phases = {n: round(float(v) * 1e3, 2) for n, v in zip(names, mean_ph)}  # microseconds

    # ---- end to end through the public API with host buffers (pinned), per step:
    #      H2D of points, features, grad, weights; D2H of y, grad_in, dW
    pts_p = torch.from_numpy(pts_h).pin_memory()
    X_p, W_p, G_p = X.cpu().pin_memory(), W.cpu().pin_memory(), G.cpu().pin_memory()
    y_p = torch.empty((N, C_OUT), dtype=torch.bfloat16).pin_memory()
    gi_p = torch.empty((N, C_IN), dtype=torch.bfloat16).pin_memory()
    gw_p = torch.empty((K_OFF, C_OUT, C_IN), dtype=torch.float32).pin_memory()
    h2d = pts_p.numel() * 4 + (X_p.numel() + W_p.numel() + G_p.numel()) * 2
    d2h = (y_p.numel() + gi_p.numel()) * 2 + gw_p.numel() * 4

    # Copies run on their own streams so they overlap the compute, as a user of the API
    # would do: H2D of the points first (quantize needs them), then features and weights
    # (fwd), then the output gradient (dgrad) while the coordinates and the map are built;
    # each result goes back D2H as soon as its kernel finished (y during dgrad, grad_in
    # during wgrad).  Consecutive steps are pipelined like a streaming training loop: step
    # i+1's uploads overlap step i's downloads (PCIe is full duplex); every step still moves
    # all of its own inputs and results.  84 MB cross PCIe per step, so e2e is PCIe bound.
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def e2e_step(start=None):
        if start is not None:
            h2d_s.wait_event(start)
        with torch.cuda.stream(h2d_s):
            p = pts_p.to(dev, non_blocking=True)
            ev_p = torch.cuda.Event()
            ev_p.record(h2d_s)
            x, w = (t.to(dev, non_blocking=True) for t in (X_p, W_p))
            ev_x = torch.cuda.Event()
            ev_x.record(h2d_s)
            g = G_p.to(dev, non_blocking=True)  # needed from dgrad on
            ev_g = torch.cuda.Event()
            ev_g.record(h2d_s)
        for t in (p, x, w, g):
            t.record_stream(stream)
        flush.zero_()  # L2 flush before this step's compute (inside the timed region)
        stream.wait_event(ev_p)
        c, _, _ = mk.coords_quantize(p, synthetic.ROOM_VOXEL, deferred=True)
        m = mk.kmap_build(c, c, region)
        stream.wait_event(ev_x)

        def to_host(dev_t, host_t):  # D2H on its own stream as soon as dev_t is ready
            ev = torch.cuda.Event()
            ev.record(stream)
            d2h_s.wait_event(ev)
            with torch.cuda.stream(d2h_s):
                host_t.copy_(dev_t, non_blocking=True)
            dev_t.record_stream(d2h_s)

        y = mk.conv_forward(m, x, w)
        to_host(y, y_p)  # overlaps dgrad
        stream.wait_event(ev_g)
        gin, _ = mk.conv_backward(m, g, x, w, need_gin=True, need_gw=False)
        to_host(gin, gi_p)  # overlaps wgrad
        _, gw = mk.conv_backward(m, g, x, w, need_gin=False, need_gw=True)
        if ws > 1:
            allreduce_grad(gw)
        to_host(gw, gw_p)

    # warm-up: at least W steps and 0.3 s of transfers (an idle PCIe link trains up to full
    # speed only under sustained traffic; the first e2e of a fresh process was 3-5x slower)
    tw, nw = time.time(), 0
    while nw < max(args.warmup, 3) or time.time() - tw < 0.3:
        e2e_step()
        nw += 1
        if nw % 4 == 0:
            torch.cuda.synchronize()
    stream.wait_stream(d2h_s)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        e2e_step(e0 if i == 0 else None)
    stream.wait_stream(d2h_s)  # the last results are on the host
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = float(e0.elapsed_time(e1))
    if ws > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = ws * flops_step / (e2e_ms / args.steps * 1e-3) / 1e12

    # ---- SURVEY §8(f) rows built so far, timed on the same scan (not part of the step):
    #      f1 label reduction, f2 stride-2 2^3 max / average pooling (Alg. 3/4),
    #      f4 generative output coordinates + transposed conv, f3 TS-CRF (Alg. 5)
    def timed(fn, reps=20):
        fn()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            ev[0].record(stream)
            fn()
            ev[1].record(stream)
            torch.cuda.synchronize()
            tot += ev[0].elapsed_time(ev[1])
        return tot / reps * 1e3  # us

    cq, p2r, first = mk.coords_quantize(pts, synthetic.ROOM_VOXEL)
    labs = (torch.arange(pts.shape[0], device=dev, dtype=torch.int32) // 7) % 5
    t_lab = timed(lambda: mk.coords_labels(p2r, first, labs))
    coarse = mk.coords_stride(cq, [2, 2, 2])
    mp = mk.kmap_build(cq, coarse, mk.Region(mk.HYPERCUBE, 3, 2))
    yp, am = mk.pool_forward(mp, X, mk.POOL_MAX)
    Gp = torch.ones_like(yp)
    t_pf = timed(lambda: mk.pool_forward(mp, X, mk.POOL_MAX, out=yp, argmax=am))
    t_pb = timed(lambda: mk.pool_backward(mp, Gp, mk.POOL_MAX, am))
    t_af = timed(lambda: mk.pool_forward(mp, X, mk.POOL_AVG, out=yp))
    pool_bytes = mp.n_in * C_IN * 2 + mp.n_out * C_IN * (2 + 4)  # x read, y + argmax written
    # f4: generative upsampling of the stride-2 set back to stride 1 ({0,1}^3) + its convT
    r2 = mk.Region(mk.HYPERCUBE, 3, 2)
    t_exp = timed(lambda: mk.coords_expand(coarse, r2, [1, 1, 1]), reps=10)
    up = mk.coords_expand(coarse, r2, [1, 1, 1])
    mup = mk.kmap_build(coarse, up, r2, transposed=True)
    Yc = torch.ones((coarse.n, C_IN), dtype=torch.bfloat16, device=dev)
    Wt = torch.full((8, C_OUT, C_IN), 0.01, dtype=torch.bfloat16, device=dev)
    t_gen = timed(lambda: mk.conv_transpose_forward(mup, Yc, Wt))
    # f3: TS-CRF mean-field inference (3 iterations, 16 classes) on the scan lifted to 7D
    #     (x, y, z, r, g, b, t) with a synthetic colour per 10 cm cell, 7D hypercross (15)
    ck = cq.export()
    col = (torch.div(ck[:, :3], 5, rounding_mode="floor") % 7).to(torch.int32)
    c7rows = torch.cat([ck[:, :3], col, torch.zeros_like(ck[:, :1]), ck[:, 3:]], dim=1)
    c7 = mk.coords_create(c7rows)
    m7 = mk.kmap_build(c7, c7, mk.Region(mk.HYPERCROSS, 7, 3))
    phi = torch.randn((c7.n, 16), device=dev)
    W7 = torch.randn((15, 16, 16), device=dev) * 0.1
    t_crf = timed(lambda: mk.crf_infer(m7, phi, W7, 3), reps=10)
    gq7 = torch.randn_like(phi)
    t_crf_bwd = timed(lambda: mk.crf_backward(m7, phi, W7, 3, gq7), reps=10)
    # f4: MinkUNet-shaped layer stack with cached coordinate sets and fused
    #     BN/ReLU/residual epilogues, bf16: stem conv, residual block (stride 1, 64 ch),
    #     stride-2 down conv 2^3 (64 -> 128), residual block (stride 2, 128 ch), transposed up
    #     conv 2^3 (128 -> 64) back onto the cached stride-1 set with an additive skip from
    #     the first block (R27).  Timed with the coordinate / map construction and without it.
    def bn(c, seed):
        g = torch.Generator(device="cpu").manual_seed(seed)
        return (torch.rand(c, generator=g) * 0.5 + 0.75).to(dev), (torch.rand(c, generator=g) - 0.5).to(dev)
    Ws = {k: (torch.randn(shape, device=dev) * (2.0 / (shape[0] * shape[2])) ** 0.5).to(torch.bfloat16)
          for k, shape in {"stem": (27, 64, 64), "b0a": (27, 64, 64), "b0b": (27, 64, 64), "down": (8, 128, 64),
                           "b1a": (27, 128, 128), "b1b": (27, 128, 128), "up": (8, 64, 128)}.items()}
    Bs = {k: bn(W.shape[1], i) for i, (k, W) in enumerate(Ws.items())}
    r3, r2 = mk.Region(mk.HYPERCUBE, 3, 3), mk.Region(mk.HYPERCUBE, 3, 2)

    def unet_maps(c0):
        c1 = mk.coords_stride(c0, [2, 2, 2])
        return (mk.kmap_build(c0, c0, r3), mk.kmap_build(c0, c1, r2), mk.kmap_build(c1, c1, r3),
                mk.kmap_build(c1, c0, r2, transposed=True))

    def unet_layers(maps, x):
        m0, md, m1, mu = maps
        f = lambda m, h, k, **kw: mk.conv_forward(m, h, Ws[k], scale=Bs[k][0], shift=Bs[k][1], **kw)  # noqa: E731
        h = f(m0, x, "stem", relu=True)
        s0 = f(m0, f(m0, h, "b0a", relu=True), "b0b", residual=h, relu=True)
        h = f(md, s0, "down", relu=True)
        h = f(m1, f(m1, h, "b1a", relu=True), "b1b", residual=h, relu=True)
        return mk.conv_transpose_forward(mu, h, Ws["up"], scale=Bs["up"][0], shift=Bs["up"][1], residual=s0,
                                         relu=True)
    maps = unet_maps(cq)
    unet_flops = 2.0 * sum(m.n_pairs * W.shape[1] * W.shape[2] for m, W in (
        (maps[0], Ws["stem"]), (maps[0], Ws["b0a"]), (maps[0], Ws["b0b"]), (maps[1], Ws["down"]),
        (maps[2], Ws["b1a"]), (maps[2], Ws["b1b"]), (maps[3], Ws["up"])))
    t_unet_layers = timed(lambda: unet_layers(maps, X))
    t_unet_all = timed(lambda: unet_layers(unet_maps(mk.coords_quantize(pts, synthetic.ROOM_VOXEL, return_maps=False)),
                                           X), reps=10)
    extras = {
        "unet_stack_layers_us": round(t_unet_layers, 2), "unet_stack_with_maps_us": round(t_unet_all, 2),
        "unet_stack_tflops": round(unet_flops / (t_unet_layers * 1e-6) / 1e12, 2),
        "unet_stack_rows": [int(maps[0].n_out), int(maps[2].n_out)],
        "labels_us": round(t_lab, 2), "labels_mpts": round(pts.shape[0] / t_lab, 1),
        "maxpool2_fwd_us": round(t_pf, 2), "maxpool2_bwd_us": round(t_pb, 2), "avgpool2_fwd_us": round(t_af, 2),
        "maxpool2_fwd_gbs": round(pool_bytes / (t_pf * 1e-6) / 1e9, 1),
        "pool_rows": [int(mp.n_in), int(mp.n_out)],
        "expand_us": round(t_exp, 2), "generative_convT_us": round(t_gen, 2), "expand_rows": int(up.n),
        "crf7d_3iter_us": round(t_crf, 2), "crf7d_3iter_backward_us": round(t_crf_bwd, 2), "crf_nodes": int(c7.n), "crf_pairs": int(m7.n_pairs),
    }

    # ---- roofline of the dominant kernel (largest phase among the conv kernels / map build)
    pk = peaks()
    conv_ph = {"conv_fwd": mean_ph[2], "conv_dgrad": mean_ph[3], "conv_wgrad": mean_ph[4]}
    dom = max(conv_ph, key=conv_ph.get)
    dom_ms = float(conv_ph[dom])
    bytes_alg = N * C_IN * 2 + N * C_OUT * 2 + 8 * M + K_OFF * C_IN * C_OUT * 2
    ai = flops_pass / bytes_alg
    ridge = pk["bf16_tflops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    traffic = None
    summ = ROOT / "profiles" / "ncu_summary.json"
    if summ.exists():
        try:
            traffic = json.loads(summ.read_text()).get("dram_bytes_per_launch", {}).get(dom)
        except (ValueError, AttributeError):
            traffic = None
    if ai >= ridge:
        achieved = flops_pass / (dom_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": round(achieved, 2), "peak": pk["bf16_tflops"], "unit": "TFLOP/s"}
    else:
        achieved = bytes_alg / (dom_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s"}
    roof.update({"frac": round(roof["achieved"] / roof["peak"], 4), "traffic": traffic, "kernel": dom,
                 "kernel_us": round(dom_ms * 1e3, 2), "algorithmic_flops": flops_pass,
                 "algorithmic_bytes": bytes_alg, "arith_intensity": round(ai, 1), "peak_source": pk["source"]})
    # The bound that actually binds the gather-GEMMs: L2 -> SM traffic of the
    # random row gathers (ncu l1tex__m_xbar2l1tex_read_bytes per launch, profiles/) over the
    # same live phase time, against the gather ceiling measured by tools/ubench_gather.cu
    # (cp.async warp-stage gathers of the same 150k x 128 B table, profiles/ubench_gather_r01.txt).
    gather = None
    ub = ROOT / "profiles" / "ubench_gather_r01.txt"
    try:
        l2sm = json.loads(summ.read_text())["kernels"][dom]["l2_to_sm_bytes"] if summ.exists() else None
        ceil = max(float(ln.split("TB/s")[0].split()[-1]) for ln in ub.read_text().splitlines()
                   if ln.startswith("cp.async warp-stage")) if ub.exists() else None
    except (ValueError, KeyError, AttributeError):
        l2sm, ceil = None, None
    if l2sm and ceil:
        ach = l2sm / (dom_ms * 1e-3) / 1e12
        gather = {"bound": "l2_gather", "achieved": round(ach, 2), "peak": ceil, "unit": "TB/s",
                  "frac": round(ach / ceil, 4), "bytes_per_launch": l2sm, "kernel": dom,
                  "source": "ncu l2->sm bytes (profiles/ncu_summary.json) / live phase time; "
                            "ceiling tools/ubench_gather.cu"}

    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": step_config(N, M, int(pts_h.shape[0]), args.seed, ws),
        "phases_us": phases,
        "conv_tflops": round(flops_step / ((mean_ph[2] + mean_ph[3] + mean_ph[4]) * 1e-3) / 1e12, 3),
        "kmap_mpts": round(N / (mean_ph[1] * 1e-3) / 1e6, 2),
        "quantize_mpts": round(pts_h.shape[0] / (mean_ph[0] * 1e-3) / 1e6, 2),
        "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_ms / args.steps, 4)},
        "gpu_launches": int(launches),
        "extras_f1_f4": extras,
        "roofline": roof,
        "roofline_gather": gather,
        "clocks": clocks,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(pts_h, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- CPU oracle
def oracle_sample(pts_h, budget_s):
    """The oracle, as it stands (single thread), on a bounded sample of the configs[1] step:
    quantize + kernel map on the full scan, then fwd + dgrad + wgrad on the pairs of the
    first k offsets, k grown until the budget is used.  Returns (flops, seconds, sample)."""
    import oracle
    import synthetic
    t0 = time.perf_counter()
    coords, _, _ = oracle.quantize(pts_h, synthetic.ROOM_VOXEL)
    offs = oracle.region(0, 3, [3, 3, 3])
    ptr, ins, outs = oracle.kmap(coords, coords, offs)
    t_map = time.perf_counter() - t0
    N = coords.shape[0]
    X = synthetic.features(1, N, C_IN).astype(np.float64)
    W = synthetic.weights(2, K_OFF, C_OUT, C_IN).astype(np.float64)
    G = synthetic.features(3, N, C_OUT).astype(np.float64)
    flops, t_conv, k = 0.0, 0.0, 0
    while k < K_OFF and t_map + t_conv < budget_s:
        sub = (np.array([0, ptr[k + 1] - ptr[k]], np.int64), ins[ptr[k]:ptr[k + 1]], outs[ptr[k]:ptr[k + 1]])
        t1 = time.perf_counter()
        oracle.conv_forward(sub, X, W[k:k + 1], N)
        oracle.conv_dgrad(sub, G, W[k:k + 1], N)
        oracle.conv_wgrad(sub, G, X, 1)
        t_conv += time.perf_counter() - t1
        flops += 3 * 2.0 * C_IN * C_OUT * (ptr[k + 1] - ptr[k])
        k += 1
    sample = (f"configs[1] room ({pts_h.shape[0]} points, {N} voxels): oracle quantize + kernel map on the full "
              f"scan, fwd+dgrad+wgrad fp64 on the pairs of offsets 0..{k - 1} of 27")
    return flops, t_map + t_conv, sample


def cpu_baseline(pts_h, budget_s):
    flops, secs, sample = oracle_sample(pts_h, budget_s)
    return {"value": round(flops / secs / 1e12, 6), "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
            "seconds": round(secs, 2), "host_cpus": os.cpu_count()}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    pts_h = workload(args.seed)
    budget = max(2.0, min(args.cpu_seconds, 20.0))
    for _ in range(min(args.warmup, 1)):
        oracle_sample(pts_h, 1.0)
    flops, secs = 0.0, 0.0
    sample = ""
    for _ in range(args.steps):
        f, s, sample = oracle_sample(pts_h, budget / max(args.steps, 1))
        flops += f
        secs += s
    v = flops / secs / 1e12
    import oracle
    import synthetic
    coords, _, _ = oracle.quantize(pts_h, synthetic.ROOM_VOXEL)
    ptr, _, _ = oracle.kmap(coords, coords, oracle.region(0, 3, [3, 3, 3]))
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": UNIT, "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(secs / args.steps * 1e3, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": step_config(coords.shape[0], int(ptr[-1]), pts_h.shape[0], args.seed, ws),
           "cpu_baseline": {"value": round(v, 6), "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_mk(args, ws, rank, local)


if __name__ == "__main__":
    main()

"""bench.py — measures the generalized sparse convolution hot path (arXiv 1904.08755) on B200.

One step = one pass of every SURVEY.md §8(a) row over one batch of synthetic input:
quantize the float points into a coordinate hash table (a1, a2), build the kernel map
(a4, a5; for configs[3] also the strided output coordinates a3 and the transposed map), then
conv forward, input gradient and weight gradient (a6-a8; configs[3] adds the transposed
conv a9).  Inputs are resident in HBM when the timed region starts; L2 is flushed (256 MiB
write, outside the step's events) before every timed step; each step is timed with CUDA
events on the launching stream.

Workloads (--config, the index into BASELINE.json "configs"; default 4):
  0  2,000 random cells of 32^3, 3x3x3, C 16 -> 16 (integer coordinates)
  1  one ScanNet-shaped room, 2 cm voxels (~150k), 3x3x3, C 64 -> 64
  2  3-frame Synthia-shaped video, 4D, hybrid kernel (29 offsets), C 32 -> 64
  3  the room's U-Net layer pair: stride-2 2x2x2 conv 128 -> 256 (+ output coordinates)
     and its transposed conv 256 -> 128
  4  16 ScanNet-shaped rooms (b = 0..15, ~2.4M voxels), 3x3x3, C 96 -> 96, sharded by batch
     index over the ranks (LPT on |M|); NCCL all-reduce of dW in the step, NCCL all-gather
     of the outputs timed separately.  This is the configuration the metric's
     "3x3x3, ScanNet-like @1/2/4/8 GPU" names, so it is the default (strong scaling: the
     16 scans are split over N ranks).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config I] [--dtype bf16|f32]
                        [--impl mk|reference]
--gpus N > 1 without torchrun in the environment re-launches itself under
torch.distributed.run (one process per GPU, NCCL).  `--impl reference` times the CPU oracle
(oracle/; the only other place bench.py runs it) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
N_SCANS = 16  # configs[4]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mk", choices=["mk", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the other configs / f1-f4 sub-lines")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=25.0)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def maybe_self_launch(args):
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) on this node and pass rank
    0's line through."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained") or d["bf16_tflops"], "source": "measured",
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0)}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback",
            "sm_max_mhz": 1965.0}


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


# ---------------------------------------------------------------------------- workloads
DESC = {
    0: "configs[0]: 2,000 random cells of 32^3, 3x3x3 hypercube, C 16->16, create + hash + kernel map + fwd + dgrad "
       "+ wgrad",
    1: "configs[1]: ScanNet-shaped room, 2 cm voxels, 3x3x3 hypercube, C 64->64, quantize + hash + kernel map + fwd "
       "+ dgrad + wgrad",
    2: "configs[2]: Synthia-shaped 3-frame video, 4D, hybrid kernel (3^3 x temporal cross, 29 offsets), C 32->64, "
       "create + hash + kernel map + fwd + dgrad + wgrad",
    3: "configs[3]: U-Net layer pair on the ScanNet-shaped room: quantize + stride-2 output coordinates + 2x2x2 map and "
       "its transposed map, conv 128->256 and convT 256->128, each fwd + dgrad + wgrad",
    4: "configs[4]: 16 ScanNet-shaped rooms (b = 0..15), 3x3x3 hypercube, C 96->96, sharded by batch index (LPT on "
       "|M|), quantize + hash + kernel map + fwd + dgrad + wgrad + NCCL all-reduce of dW per rank; NCCL all-gather "
       "of the outputs timed separately",
}
DEFAULT_SEED = {0: 1000, 1: 2000, 2: 3000, 3: 2000, 4: 5000}


def seed_of(args, cfg):
    return args.seed if args.seed is not None else DEFAULT_SEED[cfg]


def host_inputs(cfg, seed, rank=0, ws=1):
    """Seeded host inputs of a workload (synthetic/: no method arithmetic).  Returns a dict:
    kind 'points' (float points [+ batch], quantized in the step) or 'rows' (integer rows,
    created in the step)."""
    import synthetic
    if cfg == 0:
        return {"kind": "rows", "rows": synthetic.random_cells(seed, 2000, 32), "D": 3}
    if cfg in (1, 3):
        return {"kind": "points", "points": synthetic.room_points(seed), "batch": None, "voxel": synthetic.ROOM_VOXEL}
    if cfg == 2:
        return {"kind": "video", "points": synthetic.video_points(seed), "voxel": synthetic.VIDEO_VOXEL}
    pts, bat = synthetic.rooms_batch(seed, N_SCANS)
    return {"kind": "points", "points": pts, "batch": bat, "voxel": synthetic.ROOM_VOXEL}


class Workload:
    """Device-resident inputs and the step of one configuration on one rank."""

    def __init__(self, cfg, args, dev, rank, ws, dtype):
        import torch

        import paper_1904_08755_b200 as mk
        import synthetic
        from paper_1904_08755_b200.dist import lpt_assign, rank_points
        self.mk, self.torch, self.cfg, self.dev, self.ws, self.rank = mk, torch, cfg, dev, ws, rank
        self.tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        seed = seed_of(args, cfg)
        self.seed = seed
        inp = host_inputs(cfg, seed)
        self.scans = None
        self._bat_e2e = None
        if cfg == 4:  # LPT shard plan on per-scan |M| (setup, the same on every rank)
            pts_all, bat_all = inp["points"], inp["batch"]
            costs = []
            r3 = mk.Region(mk.HYPERCUBE, 3, 3)
            for b in range(N_SCANS):
                sel = bat_all == b
                cb = mk.coords_quantize(torch.from_numpy(pts_all[sel]).to(dev), inp["voxel"], return_maps=False)
                costs.append(float(mk.kmap_build(cb, cb, r3).n_pairs))
            self.scans = lpt_assign(costs, ws)[rank]
            p, b = rank_points(pts_all, bat_all, self.scans)
            inp = dict(inp, points=p, batch=b)
        if inp["kind"] == "video":  # 4D rows (x, y, z, t; b = 0), integer input of the step
            pts, fr = inp["points"]
            c3 = mk.coords_quantize(torch.from_numpy(pts).to(dev), inp["voxel"], torch.from_numpy(fr).to(dev),
                                    return_maps=False)
            r = c3.export()
            rows = torch.cat([r[:, :3], r[:, 3:4], torch.zeros_like(r[:, :1])], dim=1).cpu().numpy()
            inp = {"kind": "rows", "rows": rows, "D": 4}
        self.inp = inp
        if inp["kind"] == "points":
            self.h_pts = inp["points"]
            self.h_bat = inp["batch"]
            self.pts = torch.from_numpy(self.h_pts).to(dev)
            self.bat = None if self.h_bat is None else torch.from_numpy(self.h_bat).to(dev)
            self.voxel = inp["voxel"]
            self.n_points = int(self.h_pts.shape[0])
        else:
            self.h_rows = inp["rows"]
            self.rows = torch.from_numpy(self.h_rows).to(dev)
            self.n_points = int(self.h_rows.shape[0])
        if cfg == 2:
            self.region = mk.Region(mk.HYBRID, 4, 3)
        elif cfg == 3:
            self.region = mk.Region(mk.HYPERCUBE, 3, 2)
        else:
            self.region = mk.Region(mk.HYPERCUBE, 3, 3)
        # one untimed pass fixes the sizes
        c = self.coords(self.pts if inp["kind"] == "points" else self.rows)
        self.N = c.n
        if cfg == 3:
            coarse = mk.coords_stride(c, [2, 2, 2])
            md = mk.kmap_build(c, coarse, self.region)
            self.N_coarse = coarse.n
            self.M = md.n_pairs
            self.layers = [("down", 128, 256, md.n_in, md.n_out), ("up", 256, 128, md.n_out, md.n_in)]
        else:
            m = mk.kmap_build(c, c, self.region)
            self.M = m.n_pairs
            cin, cout = {0: (16, 16), 1: (64, 64), 2: (32, 64), 4: (96, 96)}[cfg]
            self.layers = [("", cin, cout, self.N, self.N)]
        K = 8 if cfg == 3 else (29 if cfg == 2 else 27)
        self.K = K
        self.feats = {}
        for i, (nm, cin, cout, n_in, n_out) in enumerate(self.layers):
            # features of the rank's rows: the global row generator sliced to this rank's rows
            # (configs[4]: every rank draws its own rows' features with the same recipe)
            X = synthetic.features(1 + 10 * i + 100 * rank, n_in, cin)
            W = synthetic.weights(2 + 10 * i, K, cout, cin)
            G = synthetic.features(3 + 10 * i + 100 * rank, n_out, cout)
            self.feats[nm] = tuple(torch.from_numpy(a).to(dev).to(self.tdt) for a in (X, W, G))
        self.flops_layer = {nm: 2.0 * cin * cout * self.M for (nm, cin, cout, _, _) in self.layers}
        self.flops_step = 3.0 * sum(self.flops_layer.values())
        del c

    # -- the steps of the path
    def coords(self, src, deferred=False):
        mk = self.mk
        if self.inp["kind"] == "points":
            return mk.coords_quantize(src, self.voxel, self.bat if src is self.pts else self._bat_e2e,
                                      return_maps=False, deferred=deferred)
        return mk.coords_create(src)

    def phases(self):
        return (["quantize" if self.inp["kind"] == "points" else "create"]
                + (["stride", "kmap"] if self.cfg == 3 else ["kmap"])
                + [f"{p}{('_' + nm) if nm else ''}" for (nm, *_r) in self.layers for p in ("conv_fwd", "conv_dgrad",
                                                                                          "conv_wgrad")]
                + (["allreduce_dW"] if self.ws > 1 else []))

    def step(self, mark, src=None, feats=None, on_result=None):
        """One pass of the path; mark(i) records event i (phase boundaries).  src / feats
        override the resident inputs (the e2e step); on_result(name, tensor) is called as
        each result is produced."""
        mk = self.mk
        from paper_1904_08755_b200.dist import allreduce_grad
        feats = feats or self.feats
        i = 0
        mark(i)
        c = self.coords(self.pts if (src is None and self.inp["kind"] == "points") else
                        (self.rows if src is None else src), deferred=self.inp["kind"] == "points")
        i += 1
        mark(i)
        if self.cfg == 3:
            coarse = mk.coords_stride(c, [2, 2, 2])
            i += 1
            mark(i)
            maps = {"down": mk.kmap_build(c, coarse, self.region), "up": mk.kmap_build(coarse, c, self.region,
                                                                                        transposed=True)}
        else:
            maps = {"": mk.kmap_build(c, c, self.region)}
        i += 1
        mark(i)
        outs = {}
        for (nm, cin, cout, n_in, n_out) in self.layers:
            X, W, G = feats[nm]
            m = maps[nm]
            fwd = mk.conv_transpose_forward if nm == "up" else mk.conv_forward
            bwd = mk.conv_transpose_backward if nm == "up" else mk.conv_backward
            y = fwd(m, X, W)
            i += 1
            mark(i)
            if on_result:
                on_result("y" + nm, y)
            gin, _ = bwd(m, G, X, W, need_gin=True, need_gw=False)
            i += 1
            mark(i)
            if on_result:
                on_result("gin" + nm, gin)
            _, gw = bwd(m, G, X, W, need_gin=False, need_gw=True)
            i += 1
            mark(i)
            outs[nm] = (y, gin, gw)
        if self.ws > 1:
            for nm in outs:
                allreduce_grad(outs[nm][2])  # data-parallel weight-gradient sum (NCCL over NVLink)
            i += 1
            mark(i)
        if on_result:
            for nm in outs:
                on_result("gw" + nm, outs[nm][2])
        return outs

    # -- algorithmic work
    def map_bytes(self):
        """Compulsory bytes of quantize/create + kernel-map build (§8(d), table at its minimum
        load-1/2 capacity of 2N slots of 20 B): N_p (4 D + 4 batch) read + 4 N_p point->row
        written (quantize only) + 16 N coords written + 40 N table bytes + 16 N_out query
        coords read + 8 |M| pair bytes written (+ a3's 16 N read / 16 N_coarse written)."""
        D = 4 if self.cfg == 2 else 3
        b = 0
        if self.inp["kind"] == "points":
            b += self.n_points * (4 * D + (4 if self.h_bat is not None else 0) + 4)
        else:
            b += self.n_points * 4 * (D + 1)
        b += self.N * (16 + 40)
        if self.cfg == 3:
            b += 16 * self.N + 16 * self.N_coarse + 40 * self.N_coarse  # stride: read C_in, write C_out + its table
            b += 2 * (16 * self.N + 8 * self.M)  # the two maps
        else:
            b += 16 * self.N + 8 * self.M
        return b

    def conv_roof(self, nm, pk, dtype, t_ms):
        """Roofline of a conv launch: flops 2 C_in C_out |M|, compulsory bytes of §8(d)."""
        (_, cin, cout, n_in, n_out) = [L for L in self.layers if L[0] == nm][0]
        s = 2 if dtype == "bf16" else 4
        flops = 2.0 * cin * cout * self.M
        byts = n_in * cin * s + n_out * cout * s + 8 * self.M + self.K * cin * cout * s
        ai = flops / byts
        if dtype == "f32" and (cin % 16 or cout % 16 or os.environ.get("MK_F32_MODE") == "exact"):
            # exact FFMA path: FP32 ALU bound (148 SMs x 128 lanes x 2 flop x clock)
            peak = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
            ach = flops / (t_ms * 1e-3) / 1e12
            return {"bound": "alu", "achieved": round(ach, 2), "peak": round(peak, 1), "unit": "TFLOP/s",
                    "frac": round(ach / peak, 4), "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x max clock"}
        if dtype == "f32":
            # fp32 on the bf16 tensor cores by three-way operand splitting (conv_split.cu): six
            # bf16 products per fp32 product, so the fp32 peak is the bf16 peak / 6
            peak = pk["bf16_tflops_sustained"] / 6.0
            ach = flops / (t_ms * 1e-3) / 1e12
            return {"bound": "tensor", "achieved": round(ach, 2), "peak": round(peak, 1), "unit": "TFLOP/s",
                    "frac": round(ach / peak, 4), "algorithmic_flops": flops,
                    "peak_source": pk["source"] + " sustained bf16 / 6 (bf16x3 split: 6 bf16 products per fp32 product)"}
        ridge = pk["bf16_tflops_sustained"] * 1e12 / (pk["hbm_gbs"] * 1e9)
        if ai >= ridge:
            ach = flops / (t_ms * 1e-3) / 1e12
            return {"bound": "tensor", "achieved": round(ach, 2), "peak": pk["bf16_tflops_sustained"],
                    "unit": "TFLOP/s", "frac": round(ach / pk["bf16_tflops_sustained"], 4),
                    "algorithmic_flops": flops, "algorithmic_bytes": byts, "arith_intensity": round(ai, 1),
                    "peak_source": pk["source"] + " (sustained bf16: the kernel is timed inside a long step)"}
        ach = byts / (t_ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / pk["hbm_gbs"], 4), "algorithmic_flops": flops, "algorithmic_bytes": byts,
                "arith_intensity": round(ai, 1), "peak_source": pk["source"]}


def time_steps(w, steps, warmup, stream, flush, sync_ranks=None):
    """Warm-up, then `steps` timed steps (L2 flushed before each, outside its events).
    Returns (per-phase ms [steps][phases], launches in the timed region)."""
    import torch
    n_ph = len(w.phases())
    for _ in range(warmup):
        w.step(lambda i: None)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ph + 1)] for _ in range(steps)]
    launches0 = w.mk.kernel_launch_count()
    import gc
    gc.collect()
    gc.disable()  # a collector pass inside a step would stall the host while the GPU drains
    if sync_ranks:
        sync_ranks()
    torch.cuda.synchronize()
    for s in range(steps):
        flush.zero_()
        w.step(lambda i, e=evs[s]: e[i].record(stream))
    torch.cuda.synchronize()
    gc.enable()
    if sync_ranks:
        sync_ranks()
    launches = w.mk.kernel_launch_count() - launches0
    ph = np.array([[evs[s][j].elapsed_time(evs[s][j + 1]) for j in range(n_ph)] for s in range(steps)])
    if os.environ.get("MK_BENCH_STEPS"):  # development: per-step phase times (us) on stderr
        for s in range(steps):
            print("step", s, " ".join(f"{v * 1e3:.0f}" for v in ph[s]), file=sys.stderr)
    return ph, launches


def e2e_measure(w, steps, warmup, stream, flush, sync_ranks=None):
    """The same step through the public API with host buffers: every step uploads its inputs
    from pinned host memory (points [+ batch] or rows, X, W, G) and downloads its results (y,
    grad_in, dW), on copy streams that overlap the compute as a user would; consecutive steps
    are pipelined (step i+1's uploads overlap step i's downloads; PCIe is full duplex).  One
    pair of events brackets all steps.  Returns (ms per step, h2d bytes, d2h bytes)."""
    import torch
    dev = w.dev
    if w.inp["kind"] == "points":
        src_h = [torch.from_numpy(w.h_pts).pin_memory()] + (
            [torch.from_numpy(w.h_bat).pin_memory()] if w.h_bat is not None else [])
    else:
        src_h = [torch.from_numpy(w.h_rows).pin_memory()]
    feats_h = {nm: tuple(t.cpu().pin_memory() for t in f) for nm, f in w.feats.items()}
    res_h = {}
    for (nm, cin, cout, n_in, n_out) in w.layers:
        res_h["y" + nm] = torch.empty((n_out, cout), dtype=w.tdt).pin_memory()
        res_h["gin" + nm] = torch.empty((n_in, cin), dtype=w.tdt).pin_memory()
        res_h["gw" + nm] = torch.empty((w.K, cout, cin), dtype=torch.float32).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in src_h) + sum(
        t.numel() * t.element_size() for f in feats_h.values() for t in f)
    d2h = sum(t.numel() * t.element_size() for t in res_h.values())
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def one(start=None):
        if start is not None:
            h2d_s.wait_event(start)
        with torch.cuda.stream(h2d_s):
            src = [t.to(dev, non_blocking=True) for t in src_h]
            ev_src = torch.cuda.Event()
            ev_src.record(h2d_s)
            feats = {nm: tuple(t.to(dev, non_blocking=True) for t in f) for nm, f in feats_h.items()}
            ev_f = torch.cuda.Event()
            ev_f.record(h2d_s)
        for t in src + [t for f in feats.values() for t in f]:
            t.record_stream(stream)
        flush.zero_()  # L2 flush before this step's compute (inside the timed region)
        stream.wait_event(ev_src)
        if w.inp["kind"] == "points":
            w._bat_e2e = src[1] if len(src) > 1 else None
            s0 = src[0]
        else:
            s0 = src[0]
        def on_result(name, t):
            ev = torch.cuda.Event()
            ev.record(stream)
            d2h_s.wait_event(ev)
            with torch.cuda.stream(d2h_s):
                res_h[name].copy_(t, non_blocking=True)
            t.record_stream(d2h_s)

        stream.wait_event(ev_f)
        w.step(lambda i: None, src=s0, feats=feats, on_result=on_result)

    tw, nw = time.time(), 0
    while nw < max(warmup, 3) or time.time() - tw < 0.3:
        one()
        nw += 1
        if nw % 4 == 0:
            torch.cuda.synchronize()
    stream.wait_stream(d2h_s)
    torch.cuda.synchronize()
    if sync_ranks:
        sync_ranks()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(steps):
        one(e0 if s == 0 else None)
    stream.wait_stream(d2h_s)
    e1.record(stream)
    torch.cuda.synchronize()
    return float(e0.elapsed_time(e1)) / steps, int(h2d), int(d2h)


def summarize(w, ph, pk, dtype):
    """Phase means, conv TFLOP/s, map Mpts/s and the two rooflines of one workload."""
    names = w.phases()
    mean = ph.mean(axis=0)
    phases = {n: round(float(v) * 1e3, 2) for n, v in zip(names, mean)}
    conv_names = [n for n in names if n.startswith("conv_")]
    conv_ms = {n: float(mean[names.index(n)]) for n in conv_names}
    dom = max(conv_ms, key=conv_ms.get)
    nm = dom.split("_", 2)[2] if dom.count("_") >= 2 else ""
    roof = w.conv_roof(nm, pk, dtype, conv_ms[dom])
    roof.update({"kernel": dom, "kernel_us": round(conv_ms[dom] * 1e3, 2), "traffic": ncu_traffic(w.cfg, dom)})
    build_ms = sum(float(mean[names.index(n)]) for n in names if n in ("quantize", "create", "stride", "kmap"))
    mb = w.map_bytes()
    ach = mb / (build_ms * 1e-3) / 1e9
    map_roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / pk["hbm_gbs"], 4), "algorithmic_bytes": int(mb), "phases": "quantize/create + "
                "stride + kmap", "time_us": round(build_ms * 1e3, 2), "traffic": ncu_traffic(w.cfg, "map_build"),
                "peak_source": pk["source"]}
    conv_total = sum(conv_ms.values())
    # the gather bound of the dominant conv kernel: rows gathered per pair (fwd: C_in, dgrad:
    # C_out, wgrad: both) against the random 128-byte-row gather ceiling measured on this GPU
    # (tools/ubench_ldgsts.cu, profiles/ubench_ldgsts_r02.txt: 10.64 TB/s with 12 warps/SM)
    (_, cin, cout, _n_in, _n_out) = [L for L in w.layers if L[0] == nm][0]
    esz = 2 if dtype == "bf16" else 4
    per_pair = {"conv_fwd": cin, "conv_dgrad": cout, "conv_wgrad": cin + cout}[dom.split("_", 2)[0] + "_" +
                                                                               dom.split("_", 2)[1]] * esz
    gb = per_pair * w.M
    gach = gb / (conv_ms[dom] * 1e-3) / 1e12
    gather = {"bound": "l2_gather", "achieved": round(gach, 2), "peak": GATHER_PEAK_TBS, "unit": "TB/s",
              "frac": round(gach / GATHER_PEAK_TBS, 4), "gathered_bytes": int(gb), "kernel": dom,
              "peak_source": "builder-measured random 128-byte row gather ceiling (tools/ubench_ldgsts.cu)"}
    return {
        "phases_us": phases,
        "conv_tflops": round(w.flops_step / (conv_total * 1e-3) / 1e12, 3),
        "kmap_mpts": round(w.N / (build_ms * 1e-3) / 1e6, 2),
        "gprobes_per_s": round(w.N * w.K / (build_ms * 1e-3) / 1e9, 2),
        "roofline": roof,
        "roofline_map_build": map_roof,
        "roofline_gather": gather,
    }


NCU_SUMMARY = {4: "ncu_summary_r02s3b.json", 1: "ncu_summary_r02s3b_c1.json"}
GATHER_PEAK_TBS = 10.64
MAP_KERNELS = ("quant_insert", "quant_rank", "kmap_probe", "kmap_emit", "kmap_sort")


def ncu_traffic(cfg, kernel):
    """DRAM bytes (read + write) per launch of a kernel of this workload from the committed
    ncu capture (tools/ncu_profile.sh: --set full --cache-control all, i.e. cold L2 as in the
    flushed bench step), or None.  "map_build" sums the map-build kernels' captures."""
    name = NCU_SUMMARY.get(cfg)
    p = ROOT / "profiles" / name if name else None
    if p is None or not p.exists():
        return None
    try:
        d = json.loads(p.read_text()).get("dram_bytes_per_launch", {})
        if kernel == "map_build":
            v = [d.get(k) for k in MAP_KERNELS]
            return None if any(x is None for x in v) else int(sum(v))
        x = d.get(kernel)
        return None if x is None else int(x)
    except (ValueError, AttributeError):
        return None


# ---------------------------------------------------------------------------- GPU arm
def run_mk(args, ws, rank, local):
    import torch
    import torch.distributed as dist

    import paper_1904_08755_b200 as mk
    from paper_1904_08755_b200.dist import RowGather

    # MK_DIST_BACKEND=gloo (development): ranks may share GPUs (device = local rank modulo the
    # visible devices) to exercise the multi-rank path where only one GPU is available
    backend = os.environ.get("MK_DIST_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    # configs[0]-[3] are single-scan workloads: under N > 1 every rank runs its own replica
    # (weak scaling, no collective other than the dW all-reduce); configs[4] is sharded
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    sync = (lambda: dist.barrier()) if ws > 1 else None
    pk = peaks()

    w = Workload(args.config, args, dev, rank, ws, args.dtype)
    sampler = ClockSampler(local_dev)
    sampler.start()
    time.sleep(0.3)
    t0 = time.time()
    ph, launches = time_steps(w, args.steps, args.warmup, stream, flush, sync)
    t1 = time.time()
    clocks = sampler.stop(t0, t1)
    total_ms = float(ph.sum())
    flops_rank = w.flops_step
    if ws > 1:
        t = torch.tensor([total_ms, flops_rank], dtype=torch.float64, device=dev)
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        total_ms, flops_all = float(tmax[0].item()), float(tsum[1].item())
    else:
        flops_all = flops_rank
    ms_per_step = total_ms / args.steps
    value = flops_all / (ms_per_step * 1e-3) / 1e12
    summ = summarize(w, ph, pk, args.dtype)
    if ws > 1:  # the committed ncu captures are of the one-GPU workload
        summ["roofline"]["traffic"] = None
        summ["roofline_map_build"]["traffic"] = None

    # ---- output all-gather (configs[4]; north star: "NCCL all-gather of outputs"), timed
    #      separately from the compute phase with events, max over ranks
    allgather = None
    if ws > 1:
        y = list(w.step(lambda i: None).values())[0][0]
        g = RowGather(y.shape[0], y.shape[1], y.dtype, dev)
        for _ in range(3):
            g(y)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            g(y)
        e1.record(stream)
        torch.cuda.synchronize()
        ag_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
        dist.all_reduce(ag_ms, op=dist.ReduceOp.MAX)
        ag = float(ag_ms.item())
        size = g.bytes_per_call  # NCCL convention: algbw = total bytes / t, busbw = algbw (N-1)/N
        allgather = {"ms": round(ag, 4), "bytes_per_rank_received": size, "algbw_gbs": round(size / (ag * 1e-3) / 1e9, 1),
                     "busbw_gbs": round(size / (ag * 1e-3) / 1e9 * (ws - 1) / ws, 1),
                     "padded_rows_per_rank": g.n_max, "rows_per_rank": g.sizes,
                     "step_plus_allgather_ms": round(ms_per_step + ag, 4)}

    e2e = None
    if not args.no_e2e:
        e2e_ms, h2d, d2h = e2e_measure(w, args.steps, args.warmup, stream, flush, sync)
        if ws > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": round(flops_all / (e2e_ms * 1e-3) / 1e12, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4)}

    n_rows = w.N
    M_rank = w.M
    if ws > 1:
        t = torch.tensor([n_rows, M_rank, w.n_points], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        n_all, M_all, p_all = (int(x) for x in t.tolist())
    else:
        n_all, M_all, p_all = n_rows, M_rank, w.n_points
    config = {"workload": DESC[args.config], "voxels": n_all, "pairs": M_all, "points": p_all,
              "voxels_rank0": n_rows, "pairs_rank0": M_rank, "seed": w.seed,
              "parallelism": f"batch-index dp{ws}" + (f" (rank 0 scans {w.scans})" if w.scans is not None else ""),
              "l2": "flushed before every timed step (256 MiB write, outside the step events); the e2e step "
                    "flushes inside its timed region"}
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong" if args.config == 4 else "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic", "config": config,
        **summ,
        "allgather": allgather,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if rank == 0 and ws == 1 and not args.no_extras:
        out["other_configs"] = other_configs(args, dev, stream, flush, pk)
        out["extras_f1_f4"] = extras(dev, stream, flush)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config, w.seed, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def other_configs(args, dev, stream, flush, pk):
    """configs[1]-[3] (and [4] when the headline is another config) at N = 1, 10 steps each:
    phases, TFLOP/s and both rooflines (the same step code and timing rules as the headline)."""
    out = {}
    for cfg in (1, 2, 3, 4):
        if cfg == args.config:
            continue
        w = Workload(cfg, args, dev, 0, 1, args.dtype)
        ph, launches = time_steps(w, 10, 3, stream, flush)
        ms = float(ph.sum()) / 10
        d = {"workload": DESC[cfg], "value": round(w.flops_step / (ms * 1e-3) / 1e12, 3), "unit": UNIT,
             "ms_per_step": round(ms, 4), "voxels": w.N, "pairs": w.M, "gpu_launches": int(launches)}
        d.update(summarize(w, ph, pk, args.dtype))
        out[f"configs[{cfg}]"] = d
        del w
    return out


def extras(dev, stream, flush):
    """SURVEY §8(f) rows f1-f4 on the configs[1] room, outside the step (not the headline)."""
    import torch

    import paper_1904_08755_b200 as mk
    import synthetic

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

    pts = torch.from_numpy(synthetic.room_points(2000)).to(dev)
    X = torch.from_numpy(synthetic.features(1, 1, 64)).to(dev)  # placeholder, resized below
    cq, p2r, first = mk.coords_quantize(pts, synthetic.ROOM_VOXEL)
    X = torch.from_numpy(synthetic.features(1, cq.n, 64)).to(dev).to(torch.bfloat16)
    labs = (torch.arange(pts.shape[0], device=dev, dtype=torch.int32) // 7) % 5
    t_lab = timed(lambda: mk.coords_labels(p2r, first, labs))
    coarse = mk.coords_stride(cq, [2, 2, 2])
    r2, r3 = mk.Region(mk.HYPERCUBE, 3, 2), mk.Region(mk.HYPERCUBE, 3, 3)
    mp = mk.kmap_build(cq, coarse, r2)
    yp, am = mk.pool_forward(mp, X, mk.POOL_MAX)
    Gp = torch.ones_like(yp)
    t_pf = timed(lambda: mk.pool_forward(mp, X, mk.POOL_MAX, out=yp, argmax=am))
    t_pb = timed(lambda: mk.pool_backward(mp, Gp, mk.POOL_MAX, am))
    t_af = timed(lambda: mk.pool_forward(mp, X, mk.POOL_AVG, out=yp))
    pool_bytes = mp.n_in * 64 * 2 + mp.n_out * 64 * (2 + 4)
    t_exp = timed(lambda: mk.coords_expand(coarse, r2, [1, 1, 1]), reps=10)
    up = mk.coords_expand(coarse, r2, [1, 1, 1])
    mup = mk.kmap_build(coarse, up, r2, transposed=True)
    Yc = torch.ones((coarse.n, 64), dtype=torch.bfloat16, device=dev)
    Wt = torch.full((8, 64, 64), 0.01, dtype=torch.bfloat16, device=dev)
    t_gen = timed(lambda: mk.conv_transpose_forward(mup, Yc, Wt))
    ck = cq.export()
    col = (torch.div(ck[:, :3], 5, rounding_mode="floor") % 7).to(torch.int32)
    c7 = mk.coords_create(torch.cat([ck[:, :3], col, torch.zeros_like(ck[:, :1]), ck[:, 3:]], dim=1))
    m7 = mk.kmap_build(c7, c7, mk.Region(mk.HYPERCROSS, 7, 3))
    phi = torch.randn((c7.n, 16), device=dev)
    W7 = torch.randn((15, 16, 16), device=dev) * 0.1
    t_crf = timed(lambda: mk.crf_infer(m7, phi, W7, 3), reps=10)

    def bn(c, seed):
        g = torch.Generator(device="cpu").manual_seed(seed)
        return (torch.rand(c, generator=g) * 0.5 + 0.75).to(dev), (torch.rand(c, generator=g) - 0.5).to(dev)
    Ws = {k: (torch.randn(shape, device=dev) * (2.0 / (shape[0] * shape[2])) ** 0.5).to(torch.bfloat16)
          for k, shape in {"stem": (27, 64, 64), "b0a": (27, 64, 64), "b0b": (27, 64, 64), "down": (8, 128, 64),
                           "b1a": (27, 128, 128), "b1b": (27, 128, 128), "up": (8, 64, 128)}.items()}
    Bs = {k: bn(W.shape[1], i) for i, (k, W) in enumerate(Ws.items())}

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
    t_unet = timed(lambda: unet_layers(maps, X))
    return {
        "unet_stack_layers_us": round(t_unet, 2), "unet_stack_tflops": round(unet_flops / (t_unet * 1e-6) / 1e12, 2),
        "labels_us": round(t_lab, 2), "maxpool2_fwd_us": round(t_pf, 2), "maxpool2_bwd_us": round(t_pb, 2),
        "avgpool2_fwd_us": round(t_af, 2), "maxpool2_fwd_gbs": round(pool_bytes / (t_pf * 1e-6) / 1e9, 1),
        "expand_us": round(t_exp, 2), "generative_convT_us": round(t_gen, 2), "crf7d_3iter_us": round(t_crf, 2),
    }


# ---------------------------------------------------------------------------- CPU oracle
def oracle_step(cfg, seed, threads, max_offsets=None):
    """The oracle, as it stands, on a bounded sample of the workload: one scan (configs[4]:
    scan 0 of the batch; configs[3]: the down layer) — quantize / create + kernel map on the
    whole scan, then fwd + dgrad + wgrad on the pairs of the first `max_offsets` offsets
    (all by default).  `threads` OpenMP threads (results are thread-count independent).
    Returns (conv flops, seconds, sample description)."""
    import oracle
    import synthetic
    oracle.set_threads(threads)
    inp = host_inputs(cfg if cfg != 4 else 1, seed)  # configs[4]: one of its rooms (seed = scan 0's)
    cin, cout = {0: (16, 16), 1: (64, 64), 2: (32, 64), 3: (128, 256), 4: (96, 96)}[cfg]
    t0 = time.perf_counter()
    if inp["kind"] == "rows":
        coords, _ = oracle.create(inp["rows"])
    elif inp["kind"] == "video":
        pts, fr = inp["points"]
        c3, _, _ = oracle.quantize(pts, inp["voxel"], fr)
        coords, _ = oracle.create(np.concatenate([c3, np.zeros((c3.shape[0], 1), np.int32)], axis=1))
    else:
        coords, _, _ = oracle.quantize(inp["points"], inp["voxel"], inp["batch"])
    D = coords.shape[1] - 1
    if cfg == 3:
        out = oracle.stride(coords, [2, 2, 2])
        offs = oracle.region(0, 3, [2, 2, 2])
    else:
        out = coords
        offs = oracle.region(2 if cfg == 2 else 0, D, [3] * D)
    ptr, ins, outs = oracle.kmap(coords, out, offs)
    t_map = time.perf_counter() - t0
    K = offs.shape[0]
    X = synthetic.features(1, coords.shape[0], cin).astype(np.float64)
    W = synthetic.weights(2, K, cout, cin).astype(np.float64)
    G = synthetic.features(3, out.shape[0], cout).astype(np.float64)
    kmax = K if max_offsets is None else min(K, max_offsets)
    sub = (np.concatenate([[0], ptr[1:kmax + 1]]).astype(np.int64), ins[:ptr[kmax]], outs[:ptr[kmax]])
    t1 = time.perf_counter()
    oracle.conv_forward(sub, X, W[:kmax], out.shape[0])
    oracle.conv_dgrad(sub, G, W[:kmax], coords.shape[0])
    oracle.conv_wgrad(sub, G, X, kmax)
    t_conv = time.perf_counter() - t1
    flops = 3 * 2.0 * cin * cout * float(ptr[kmax])
    what = "scan 0 of configs[4] (one room, C 96->96)" if cfg == 4 else f"configs[{cfg}]"
    sample = (f"{what}: oracle quantize/create + kernel map of the whole scan ({coords.shape[0]} voxels), then fp64 "
              f"fwd + dgrad + wgrad on the pairs of offsets 0..{kmax - 1} of {K} ({int(ptr[kmax])} of {int(ptr[K])} "
              f"pairs); {threads} OpenMP thread(s)")
    return flops, t_map + t_conv, sample


def cpu_baseline(cfg, seed, budget_s):
    """The oracle on the host cores (all of them, then one) on the bounded sample of
    oracle_step.  The 1-thread run covers as many offsets as fit about half the budget."""
    cores = os.cpu_count() or 1
    f, s, sample = oracle_step(cfg, seed, cores)
    out = {"value": round(f / s / 1e12, 6), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
           "seconds": round(s, 2), "host_cpus": cores}
    per_off = max(s * cores / 27.0, 1e-3)  # rough 1-thread seconds per offset
    k1 = int(max(1, min(27, (budget_s / 2) / per_off)))
    f1, s1, sample1 = oracle_step(cfg, seed, 1, max_offsets=k1)
    out["one_thread"] = {"value": round(f1 / s1 / 1e12, 6), "unit": UNIT, "cores": 1, "sample": sample1,
                         "seconds": round(s1, 2)}
    return out


def run_reference(args, ws, rank):
    """The reference arm: the oracle on this box's host cores, every step the bounded sample
    of cpu_baseline (the same workload, all cores).  Rank 0 only."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    cfg = args.config
    seed = seed_of(args, cfg)
    for _ in range(min(args.warmup, 1)):
        oracle_step(cfg, seed, cores, max_offsets=1)
    flops, secs, sample = 0.0, 0.0, ""
    for _ in range(args.steps):
        f, s, sample = oracle_step(cfg, seed, cores)
        flops += f
        secs += s
    v = flops / secs / 1e12
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": UNIT, "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(secs / args.steps * 1e3, 3),
           "higher_is_better": True, "scaling": "strong" if cfg == 4 else "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": DESC[cfg], "seed": seed, "sample": sample},
           "cpu_baseline": {"value": round(v, 6), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        ws, rank, _ = dist_env()
        run_reference(args, ws, rank)
        return
    maybe_self_launch(args)
    ws, rank, local = dist_env()
    run_mk(args, ws, rank, local)


if __name__ == "__main__":
    main()

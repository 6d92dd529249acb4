"""Host cost of the Python binding around the C calls on the quantize -> kmap path
(development tool): median microseconds of each piece over 50 repetitions."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402
from paper_1904_08755_b200 import _L, _ptr, _stream, context  # noqa: E402
import synthetic  # noqa: E402

pts = torch.from_numpy(synthetic.room_points(2000)).cuda()
region = mk.Region(mk.HYPERCUBE, 3, 3)
c, p2r, first = mk.coords_quantize(pts, synthetic.ROOM_VOXEL)
torch.cuda.synchronize()


def med(fn, reps=50):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return float(np.median(ts))


n = pts.shape[0]
ctx = context(0)
s = _stream(pts)


def c_quant():
    h = ctypes.c_void_p()
    _L.mk_coords_quantize(ctx, _ptr(pts), None, n, 3, ctypes.c_float(synthetic.ROOM_VOXEL), s, ctypes.byref(h),
                          _ptr(p2r), _ptr(first))
    _L.mk_coords_destroy(h)


r = mk.Region(mk.HYPERCUBE, 3, 3)._struct()


def c_kmap():
    h = ctypes.c_void_p()
    _L.mk_kmap_build(ctx, c._h, c._h, ctypes.byref(r), 0, s, ctypes.byref(h))
    _L.mk_kmap_destroy(h)


def coords_shell():
    o = object.__new__(mk.Coords)
    mk.Coords.__init__(o, c._h, pts.device)
    o._h = None  # not the owner


rows = {
    "torch.empty x2": lambda: (torch.empty(n, dtype=torch.int32, device="cuda"),
                               torch.empty(n, dtype=torch.int32, device="cuda")),
    "pts.to().contiguous()": lambda: pts.to(torch.float32).contiguous(),
    "_stream": lambda: _stream(pts),
    "context": lambda: context(0),
    "current_device": lambda: torch.cuda.current_device(),
    "Coords(h) info": lambda: coords_shell(),
    "first[:n]": lambda: first[:c.n],
    "C mk_coords_quantize": c_quant,
    "py coords_quantize": lambda: mk.coords_quantize(pts, synthetic.ROOM_VOXEL),
    "C mk_kmap_build (+destroy)": c_kmap,
    "py kmap_build": lambda: mk.kmap_build(c, c, region),
}
for k, fn in rows.items():
    print(f"{k:28s} {med(fn):8.1f} us")

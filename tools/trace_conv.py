"""Timeline of CTA 0 of the forward conv kernel (MK_TRACE build, tools/libmk_trace.so)."""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
os.environ["MK_LIBRARY"] = str(ROOT / "tools" / "libmk_trace.so")
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402
import synthetic  # noqa: E402

pts = torch.from_numpy(synthetic.room_points(2000)).cuda()
c, _, _ = mk.coords_quantize(pts, 0.02)
m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
X = torch.randn(c.n, 64, device="cuda").bfloat16()
W = (torch.randn(27, 64, 64, device="cuda") * 0.02).bfloat16()
for _ in range(3):
    mk.conv_forward(m, X, W)
torch.cuda.synchronize()
tr = np.zeros((4, 4096), np.uint64)
mk._L.mk_debug_trace.argtypes = [ctypes.c_void_p]
mk._L.mk_debug_trace(tr.ctypes.data)
t0 = int(tr[0][0])
prod = tr[0].astype(np.int64) - t0
mma = tr[1].astype(np.int64) - t0
epi = tr[2].astype(np.int64) - t0
unit = tr[3].astype(np.int64) - t0
n = 216
print("producer step: [t_before_empty_wait, t_after] (ns)")
for g in list(range(0, 12)) + list(range(100, 106)) + list(range(n - 4, n)):
    print(g, prod[2 * g], prod[2 * g + 1], " mma_full_ok", mma[g])
print("units (nbr wait start/end):", [(unit[2 * i], unit[2 * i + 1]) for i in range(9)])
print("epilogue tfull ok / done:", [(epi[2 * i], epi[2 * i + 1]) for i in range(9)])
d = np.diff(mma[:n])
print("mma step interval ns: median", np.median(d), "mean", d.mean(), "max", d.max())

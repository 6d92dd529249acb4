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
tr = np.zeros((4, 8192), np.uint64)
mk._L.mk_debug_trace.argtypes = [ctypes.c_void_p]
mk._L.mk_debug_trace(tr.ctypes.data)
t0 = int(tr[3][0])
P = (tr[0].astype(np.int64) - t0).reshape(-1, 4)
M = (tr[1].astype(np.int64) - t0).reshape(-1, 2)
U = (tr[3].astype(np.int64) - t0).reshape(-1, 4)
n = 90
print("step: prod[before_empty, empty_ok, issued, data_ok]  mma[wait, full_ok]")
for g in list(range(0, 20)) + list(range(100, 106)) + list(range(n - 3, n)):
    print(g, P[g].tolist(), M[g].tolist())
print("units: [start, n_empty_ok, staged]")
for u in range(0, 30):
    print(u, U[u, :3].tolist())
for name, arr in (("prod empty wait", P[:n, 1] - P[:n, 0]), ("prod issue", P[:n, 2] - P[:n, 1]),
                  ("prod data wait", P[:n, 3] - P[:n, 2]), ("mma full wait", M[:n, 1] - M[:n, 0])):
    print(f"{name:18s} median {np.median(arr):8.0f} ns  mean {arr.mean():8.0f}  max {arr.max():8.0f}")
Q = (tr[2][2000:2000 + 2 * n].astype(np.int64) - t0).reshape(-1, 2)
iss = Q[:, 0] - M[:n, 1]
com = Q[:, 1] - Q[:, 0]
nxt = M[1:n, 0] - Q[:n - 1, 1]
for name, arr in (("mma issue (after full_ok -> UMMAs issued)", iss), ("mma commit", com), ("mma loop to next wait", nxt)):
    print(f"{name:42s} median {np.median(arr):8.0f} ns  mean {arr.mean():8.0f}  max {arr.max():8.0f}")

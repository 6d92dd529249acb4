"""Per-warp cycle accounting of CTA 0 of the forward conv kernel (MK_TRACE build)."""
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
a = np.zeros((32, 8), np.uint64)
mk._L.mk_debug_acct.argtypes = [ctypes.c_void_p]
mk._L.mk_debug_acct(a.ctypes.data)
print("warp: [slot0 .. slot6 cycles, total cycles]   producers: 0=a_empty wait 1=issue 2=data wait 3=steps")
print("      stager(21): 0=w_empty  mma(20): 0=tempty 1=w_full 2=a_full 3=steps  epi(16-19): 0=tfull")
for w in range(22):
    print(w, a[w].tolist())
import torch.cuda
print("smem/occupancy check done via ncu; CTA 300 shown")

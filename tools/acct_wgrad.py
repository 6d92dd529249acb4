"""Per-warp cycle accounting of CTA 100 of the bf16 wgrad kernel (MK_TRACE build).
usage: python tools/acct_wgrad.py [1|4]   (configs[1] room C=64, or configs[4] batch C=96)"""
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

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
if cfg == 4:
    p, b = synthetic.rooms_batch(5000, 16)
    c, _, _ = mk.coords_quantize(torch.from_numpy(p).cuda(), synthetic.ROOM_VOXEL, torch.from_numpy(b).cuda())
    C = 96
else:
    c, _, _ = mk.coords_quantize(torch.from_numpy(synthetic.room_points(2000)).cuda(), synthetic.ROOM_VOXEL)
    C = 64
m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
X = torch.randn(c.n, C, device="cuda").bfloat16()
W = (torch.randn(27, C, C, device="cuda") * 0.02).bfloat16()
G = torch.randn(c.n, C, device="cuda").bfloat16()
for _ in range(3):
    mk.conv_backward(m, G, X, W, need_gin=False)
torch.cuda.synchronize()
a = np.zeros((32, 8), np.uint64)
mk._L.mk_debug_acct.argtypes = [ctypes.c_void_p]
mk._L.mk_debug_acct(a.ctypes.data)
print(f"configs[{cfg}] C={C}; cycles of CTA 100 per warp; last col = total")
print("producers: 0=slot-free wait 1=gather issue 2=own-data wait 3=steps | mma: 2=full wait 3=umma issue 4=steps 5=fence 6=commit "
      "| epi: 0=tfull wait")
for w in range(21):
    if a[w].any():
        print(w, a[w].tolist())

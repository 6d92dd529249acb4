"""Per-CTA start/end timeline of the forward conv kernel (MK_TRACE build)."""
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
a = np.zeros((4096, 4), np.uint64)
mk._L.mk_debug_cta.argtypes = [ctypes.c_void_p]
mk._L.mk_debug_cta(a.ctypes.data)
n = int((c.n + 127) // 128 + 1) // 2
a = a[:n].astype(np.int64)
t0 = a[:, 0].min()
st, en, sm, steps = a[:, 0] - t0, a[:, 1] - t0, a[:, 2], a[:, 3]
dur = en - st
print(f"CTAs {n}  kernel span {en.max()/1e3:.1f} us  dur mean {dur.mean()/1e3:.1f} med {np.median(dur)/1e3:.1f} max {dur.max()/1e3:.1f} us")
print("steps mean", steps.mean(), "max", steps.max(), " ns/step (dur/steps) median", np.median(dur / np.maximum(steps, 1)))
print("start time histogram (us):", np.histogram(st / 1e3, bins=10)[0].tolist(), np.histogram(st / 1e3, bins=10)[1].round(1).tolist())
for q in (0.1, 0.5, 0.9, 0.99):
    print(f"end time q{q}: {np.quantile(en, q)/1e3:.1f} us")
print("CTAs per SM:", np.bincount(sm).max(), np.bincount(sm).min())
order = np.argsort(-dur)[:8]
print("slowest CTAs (id, steps, start, dur us):", [(int(i), int(steps[i]), round(st[i]/1e3, 1), round(dur[i]/1e3, 1)) for i in order])

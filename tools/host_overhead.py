"""Host-side cost of each public API call on the configs[1] step (development tool).
For every call: wall time of the call itself (GPU idle before it), and the GPU time between
CUDA events placed around it, median of 20."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402
import synthetic  # noqa: E402

pts = torch.from_numpy(synthetic.room_points(2000)).cuda()
region = mk.Region(mk.HYPERCUBE, 3, 3)
c, _, _ = mk.coords_quantize(pts, synthetic.ROOM_VOXEL)
m = mk.kmap_build(c, c, region)
X = torch.randn(c.n, 64, device="cuda").bfloat16()
W = (torch.randn(27, 64, 64, device="cuda") * 0.02).bfloat16()
G = torch.randn(c.n, 64, device="cuda").bfloat16()
calls = {
    "quantize": lambda: mk.coords_quantize(pts, synthetic.ROOM_VOXEL),
    "kmap": lambda: mk.kmap_build(c, c, region),
    "fwd": lambda: mk.conv_forward(m, X, W),
    "dgrad": lambda: mk.conv_backward(m, G, X, W, need_gw=False),
    "wgrad": lambda: mk.conv_backward(m, G, X, W, need_gin=False),
}
for name, fn in calls.items():
    host, gpu, total = [], [], []
    for i in range(23):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        r = fn()
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        del r
        if i >= 3:
            host.append((t1 - t0) * 1e6)
            gpu.append(e0.elapsed_time(e1) * 1e3)
            total.append((t2 - t0) * 1e6)
    print(f"{name:9s} host call {np.median(host):8.1f} us   events {np.median(gpu):8.1f} us   wall incl. sync {np.median(total):8.1f} us")

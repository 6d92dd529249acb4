"""CUPTI timeline of one TS-CRF backward (bench extras' 7D case), development tool."""
import json
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402
import synthetic  # noqa: E402

pts = torch.from_numpy(synthetic.room_points(2000)).cuda()
cq = mk.coords_quantize(pts, synthetic.ROOM_VOXEL, return_maps=False)
ck = cq.export()
col = (torch.div(ck[:, :3], 5, rounding_mode="floor") % 7).to(torch.int32)
c7 = mk.coords_create(torch.cat([ck[:, :3], col, torch.zeros_like(ck[:, :1]), ck[:, 3:]], dim=1))
m7 = mk.kmap_build(c7, c7, mk.Region(mk.HYPERCROSS, 7, 3))
phi = torch.randn((c7.n, 16), device="cuda")
W7 = torch.randn((15, 16, 16), device="cuda") * 0.1
g = torch.randn_like(phi)
for _ in range(3):
    mk.crf_backward(m7, phi, W7, 3, g)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    mk.crf_backward(m7, phi, W7, 3, g)
    torch.cuda.synchronize()
fn = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(fn)
ev = sorted([e for e in json.load(open(fn))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")],
            key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev:
    print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f}  {e['cat'][:6]} {e['name'][:70]}")

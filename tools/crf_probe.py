"""Development: time the TS-CRF inference pieces on the configs[1] scan lifted to 7D."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402
import synthetic  # noqa: E402

pts = torch.from_numpy(synthetic.room_points(2000)).cuda()
cq, _, _ = mk.coords_quantize(pts, synthetic.ROOM_VOXEL)
ck = cq.export()
col = (torch.div(ck[:, :3], 5, rounding_mode="floor") % 7).to(torch.int32)
c7 = mk.coords_create(torch.cat([ck[:, :3], col, torch.zeros_like(ck[:, :1]), ck[:, 3:]], dim=1))
m7 = mk.kmap_build(c7, c7, mk.Region(mk.HYPERCROSS, 7, 3))
phi = torch.randn((c7.n, 16), device="cuda")
W7 = torch.randn((15, 16, 16), device="cuda") * 0.1
for _ in range(3):
    mk.crf_infer(m7, phi, W7, 3)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
for _ in range(10):
    mk.crf_infer(m7, phi, W7, 3)
e[1].record()
torch.cuda.synchronize()
print(f"crf 3 iters: {e[0].elapsed_time(e[1]) / 10 * 1e3:.1f} us (warm), nodes {c7.n}, pairs {m7.n_pairs}")

"""Forward conv time vs channel count on the configs[4] map (commit / chunk-step scaling).
usage: python tools/ab_channels.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402
import synthetic  # noqa: E402

p, b = synthetic.rooms_batch(5000, 16)
c, _, _ = mk.coords_quantize(torch.from_numpy(p).cuda(), synthetic.ROOM_VOXEL, torch.from_numpy(b).cuda())
m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for C in (32, 48, 64, 80, 96, 112, 128, 160, 192, 256):
    X = torch.randn(c.n, C, device="cuda").bfloat16()
    W = (torch.randn(27, C, C, device="cuda") * 0.02).bfloat16()
    for _ in range(2):
        mk.conv_forward(m, X, W)
    ts = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mk.conv_forward(m, X, W)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[2]
    fl = 2.0 * C * C * m.n_pairs
    print(f"C={C:3d}  fwd {t * 1e3:8.1f} us  {fl / (t * 1e-3) / 1e12:6.1f} TFLOP/s  gathered {m.n_pairs * C * 2 / (t * 1e-3) / 1e12:5.2f} TB/s",
          flush=True)

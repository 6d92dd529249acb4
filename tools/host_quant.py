"""Host-side timeline of coords_quantize (MK_HOST_TIMING) and Python overhead around it."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402
import synthetic  # noqa: E402

pts = torch.from_numpy(synthetic.room_points(2000)).cuda()
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c, p2r, first = mk.coords_quantize(pts, synthetic.ROOM_VOXEL)
    t1 = time.perf_counter()
    m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"python: quantize {1e6 * (t1 - t0):.1f} us, kmap_build {1e6 * (t2 - t1):.1f} us", file=sys.stderr)

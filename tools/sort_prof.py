"""Runs the configs[1] kernel-map build a few times (use with the MK_SORT_PROF variant)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402
import synthetic  # noqa: E402

pts = torch.from_numpy(synthetic.room_points(2000)).cuda()
c, _, _ = mk.coords_quantize(pts, synthetic.ROOM_VOXEL)
for _ in range(4):
    m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
    torch.cuda.synchronize()

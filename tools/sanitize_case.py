"""Small end-to-end case of the hot path for compute-sanitizer runs (tests/test_gpu_sanitizer.py):
quantize, kernel map (sorted rows, cooperative sort), bf16 and fp32 conv fwd/dgrad/wgrad,
strided map + pooling, transposed conv.  Exits 0; the sanitizer reports errors."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402

rng = np.random.default_rng(7)
pts = torch.from_numpy((rng.random((3000, 3)) * 2.0).astype(np.float32)).cuda()
c, p2r, first = mk.coords_quantize(pts, 0.1)
m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
for dt in (torch.bfloat16, torch.float32):
    X = torch.randn(c.n, 32, device="cuda").to(dt)
    W = (torch.randn(27, 32, 32, device="cuda") * 0.1).to(dt)
    G = torch.randn(c.n, 32, device="cuda").to(dt)
    y = mk.conv_forward(m, X, W)
    gi, gw = mk.conv_backward(m, G, X, W)
cs = mk.coords_stride(c, [2, 2, 2])
ms = mk.kmap_build(c, cs, mk.Region(mk.HYPERCUBE, 3, 2))
X = torch.randn(c.n, 32, device="cuda")
yp, arg = mk.pool_forward(ms, X, mk.POOL_MAX)
W = (torch.randn(8, 16, 32, device="cuda") * 0.1).bfloat16()
yd = mk.conv_forward(ms, X.bfloat16(), W)
mt = mk.kmap_build(cs, c, mk.Region(mk.HYPERCUBE, 3, 2), transposed=True)
yt = mk.conv_transpose_forward(mt, yd, (torch.randn(8, 32, 16, device="cuda") * 0.1).bfloat16())
torch.cuda.synchronize()
print("ok", c.n, m.n_pairs, cs.n, yt.shape)

"""Development probe: time one (C_in, C_out) bf16 conv case (GPU calls vs oracle) per line."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import oracle as orc  # noqa: E402
import paper_1904_08755_b200 as mk  # noqa: E402
import synthetic  # noqa: E402

orc.set_threads(int(sys.argv[1]) if len(sys.argv) > 1 else 16)
g = np.random.default_rng(777)
rows = np.concatenate([g.integers(-9, 9, (1500, 3)), g.integers(0, 2, (1500, 1))], axis=1).astype(np.int32)
c = mk.coords_create(torch.from_numpy(rows).cuda())
oc, _ = orc.create(rows)
okm = orc.kmap(oc, oc, orc.region(0, 3, [3, 3, 3]))
m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
for pair in sys.argv[2:]:
    cin, cout = (int(x) for x in pair.split(","))
    X = synthetic.features(cin, c.n, cin)
    W = synthetic.weights(cout, 27, cout, cin)
    G = synthetic.features(cin + cout, c.n, cout)
    Xd, Wd, Gd = (torch.from_numpy(a).cuda().bfloat16() for a in (X, W, G))
    t0 = time.time()
    y = mk.conv_forward(m, Xd, Wd, out_dtype=torch.float32)
    torch.cuda.synchronize()
    t1 = time.time()
    gin, _ = mk.conv_backward(m, Gd, Xd, Wd, need_gw=False)
    torch.cuda.synchronize()
    t2 = time.time()
    _, gw = mk.conv_backward(m, Gd, Xd, Wd, need_gin=False)
    torch.cuda.synchronize()
    t3 = time.time()
    y64 = orc.conv_forward(okm, X, W, c.n)
    gw64 = orc.conv_wgrad(okm, G, X, 27)
    t4 = time.time()
    e = np.abs(y.cpu().numpy() - y64).max() / np.abs(y64).max()
    ew = np.abs(gw.cpu().numpy() - gw64).max() / np.abs(gw64).max()
    print(f"{cin}->{cout}: fwd {t1-t0:.3f}s dgrad {t2-t1:.3f}s wgrad {t3-t2:.3f}s oracle {t4-t3:.3f}s "
          f"err fwd {e:.2e} wgrad {ew:.2e}", flush=True)

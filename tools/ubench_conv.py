"""Development micro-benchmark: time the bf16 conv kernels on the configs[1] room under the
MK_DEBUG_CONV / MK_STAGES switches (each setting in a fresh process)."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run():
    import torch
    import paper_1904_08755_b200 as mk
    import synthetic
    pts = torch.from_numpy(synthetic.room_points(2000)).cuda()
    c, _, _ = mk.coords_quantize(pts, 0.02)
    m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
    X = torch.randn(c.n, 64, device="cuda").bfloat16()
    W = (torch.randn(27, 64, 64, device="cuda") * 0.02).bfloat16()
    G = torch.randn(c.n, 64, device="cuda").bfloat16()
    for _ in range(3):
        mk.conv_forward(m, X, W)
    res = {}
    for name, fn in (("fwd", lambda: mk.conv_forward(m, X, W)),
                     ("dgrad", lambda: mk.conv_backward(m, G, X, W, need_gw=False)),
                     ("wgrad", lambda: mk.conv_backward(m, G, X, W, need_gin=False))):
        fn()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(10):
            fn()
        ev[1].record()
        torch.cuda.synchronize()
        res[name] = ev[0].elapsed_time(ev[1]) / 10 * 1e3
    print("dbg", os.environ.get("MK_DEBUG_CONV", "0"), "stages", os.environ.get("MK_STAGES", "-"),
          " ".join(f"{k}={v:.1f}us" for k, v in res.items()), f"pairs={m.n_pairs}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        run()
    else:
        settings = [a.split(":") for a in sys.argv[1:]] or [["0", ""], ["1", ""], ["2", ""], ["3", ""], ["0", "4"],
                                                            ["0", "2"]]
        for dbg, st in settings:
            env = dict(os.environ, MK_DEBUG_CONV=dbg)
            if st:
                env["MK_STAGES"] = st
            subprocess.run([sys.executable, __file__, "child"], env=env)

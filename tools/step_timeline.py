"""GPU timeline of a bench step (configs[cfg]) (development tool): kernel start/end times from
torch.profiler (CUPTI), printed relative to the step start with the idle gaps between them.
Usage: python tools/step_timeline.py [n_steps] [cfg]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1904_08755_b200 as mk  # noqa: E402
import synthetic  # noqa: E402

n_steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
import types  # noqa: E402

import bench  # noqa: E402

args = types.SimpleNamespace(seed=None)
w = bench.Workload(cfg, args, torch.device("cuda", 0), 0, 1, "bf16")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def step():
    w.step(lambda i: None)


for _ in range(5):
    flush.zero_()
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(n_steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()

import json  # noqa: E402
import os  # noqa: E402
import tempfile  # noqa: E402

fn = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(fn)
tr = json.load(open(fn))["traceEvents"]
evs = [e for e in tr if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
evs.sort(key=lambda e: e["ts"])
from collections import Counter  # noqa: E402
print("trace events:", len(tr), Counter(e.get("cat") for e in tr).most_common(12))
steps, cur = [], None
for e in evs:
    if e["cat"] == "kernel" and "fill" in e["name"].lower():
        if cur:
            steps.append(cur)
        cur = []
        continue
    if cur is not None:
        cur.append(e)
if cur:
    steps.append(cur)
for si, s in enumerate(steps):
    t0 = s[0]["ts"]
    prev = t0
    busy = 0.0
    print(f"--- step {si}: {len(s)} activities")
    for e in s:
        st, en = e["ts"], e["ts"] + e["dur"]
        gap = st - prev
        busy += e["dur"]
        print(f"{st - t0:9.1f} {e['dur']:8.1f} gap {gap:7.1f}  {e['cat'][:6]} {e['name'][:60]}")
        prev = max(prev, en)
    print(f"span {prev - t0:.1f} us, busy {busy:.1f} us, idle {prev - t0 - busy:.1f} us")

"""Development diagnostic: per-step GPU phase times and host call durations of configs[3], to
tell a host stall from a slow kernel when the conv_wgrad_down phase spikes."""
import sys
import time
import types

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

w = bench.Workload(3, types.SimpleNamespace(seed=None), torch.device("cuda", 0), 0, 1, "bf16")
names = w.phases()
st = torch.cuda.current_stream()
for s in range(60):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
    host = [0.0] * (len(names) + 1)
    torch.cuda.synchronize()

    def mark(i):
        evs[i].record(st)
        host[i] = time.perf_counter()

    w.step(mark)
    torch.cuda.synchronize()
    gpu = [evs[j].elapsed_time(evs[j + 1]) * 1e3 for j in range(len(names))]
    hst = [(host[j + 1] - host[j]) * 1e6 for j in range(len(names))]
    k = names.index("conv_wgrad_down")
    flag = "  <==" if gpu[k] > 150 else ""
    print(f"step {s:2d} gpu_wgrad_down {gpu[k]:8.0f} us host_call {hst[k]:8.0f} us | gpu " +
          " ".join(f"{g:.0f}" for g in gpu) + flag, flush=True)

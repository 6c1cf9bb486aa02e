"""torch.profiler timeline of one tuxv on C4 (builder tool): GPU busy time per
kernel and the idle gaps between launches."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04447_b200 as G  # noqa: E402

dev = torch.device("cuda", 0)
n = 20000
G1 = G.device_giid(n, 100, 41, device=dev)
G2 = G.device_giid(n, 100, 42, device=dev)
S = (G2 @ G1.T).T  # column-major (Fortran) like the reference's arrays
S /= torch.linalg.norm(S)
A = S + 1e-6 * G.device_giid(n, n, 43, device=dev)
del S
for _ in range(2):
    G.tuxv(A, 100, b=32, p=8, seed=0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    G.tuxv(A, 100, b=32, p=8, seed=0)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0, t1 = evs[0].time_range.start, evs[-1].time_range.end
busy = sum(e.time_range.end - e.time_range.start for e in evs)
print(f"GPU span {(t1 - t0) / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms, kernels {len(evs)}")
gaps = []
for a, b in zip(evs, evs[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 50:
        gaps.append((g, a.name[:50], b.name[:50]))
gaps.sort(reverse=True)
for g in gaps[:15]:
    print(f"gap {g[0] / 1e3:.3f} ms after {g[1]} before {g[2]}")
agg = {}
for e in evs:
    k = e.name[:60]
    agg[k] = agg.get(k, 0) + (e.time_range.end - e.time_range.start)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:15]:
    print(f"{v / 1e3:8.3f} ms  {k}")

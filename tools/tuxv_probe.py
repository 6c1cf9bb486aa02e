"""Where TUXV's time-to-rank-k goes on C4 (20000^2, k = 100, b = 32): libsqr's
per-class CUDA-event split plus the torch profiler's kernel list for one call
(input resident, after a warm-up)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04447_b200 as G  # noqa: E402
from paper_2008_04447_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
n = 20000
G1 = G.device_giid(n, 100, 41, device=dev)
G2 = G.device_giid(n, 100, 42, device=dev)
S = (G2 @ G1.T).T
S /= torch.linalg.norm(S)
A = S + 1e-6 * G.device_giid(n, n, 43, device=dev)
del S
for _ in range(2):
    G.tuxv(A, 100, b=32, p=8, seed=0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
G.tuxv(A, 100, b=32, p=8, seed=0)
e1.record()
e1.synchronize()
print(f"tuxv C4: {e0.elapsed_time(e1):.2f} ms", flush=True)
L = _lib.lib()
L.sqr_profile_enable(10000)
G.tuxv(A, 100, b=32, p=8, seed=0)
torch.cuda.synchronize()
for k, (ms, c) in _lib.profile_collect().items():
    if c:
        print(f"  {k:14s} {ms:8.3f} ms  {int(c)} launches")
L.sqr_profile_enable(0)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    G.tuxv(A, 100, b=32, p=8, seed=0)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))

"""Kernel-class split of trqrcp at n = 32768, k = 3328, b = 128 (the TRQRCP
half of the headline metric) and of the C4-sized trqrcp inside TUXV (builder tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04447_b200 as G  # noqa: E402
from paper_2008_04447_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()
for n, k, b in [(32768, 3328, 128), (20000, 100, 32)]:
    A = G.device_giid(n, n, 5, device=dev)
    G.trqrcp(A, k, b=b, p=8, seed=0)
    torch.cuda.synchronize()
    L.sqr_profile_enable(100000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.trqrcp(A, k, b=b, p=8, seed=0)
    e1.record()
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    L.sqr_profile_enable(0)
    tot = sum(v[0] for v in prof.values())
    print(f"n={n} k={k} b={b}: total {e0.elapsed_time(e1):.2f} ms, kernels {tot:.2f} ms",
          {kk: (round(v[0], 2), v[1]) for kk, v in prof.items() if v[1]}, flush=True)
    del A
    torch.cuda.empty_cache()

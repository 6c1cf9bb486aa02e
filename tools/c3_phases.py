"""Kernel-class split of C3 (rqrcp 100000 x 2000, b=64) (builder tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04447_b200 as G  # noqa: E402
from paper_2008_04447_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()
A = G.device_giid(100000, 2000, 3, device=dev)
G.rqrcp(A, 2000, b=64, p=8, seed=0)
torch.cuda.synchronize()
L.sqr_profile_enable(100000)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
G.rqrcp(A, 2000, b=64, p=8, seed=0)
e1.record()
torch.cuda.synchronize()
prof = _lib.profile_collect()
L.sqr_profile_enable(0)
print(f"C3 total {e0.elapsed_time(e1):.2f} ms", {k: (round(v[0], 2), v[1]) for k, v in prof.items() if v[1]})

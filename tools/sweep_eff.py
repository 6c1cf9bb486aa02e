"""Per-block efficiency of the two big sweeps in one C5 call (builder tool):
durations of every gemm_tn / gemm_nn launch longer than 200 us from the torch
profiler, against the algorithmic flops of that block's sweep."""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04447_b200 as G  # noqa: E402

dev = torch.device("cuda", 0)
n = b = None
n, b = 32768, 128
A = G.device_giid(n, n, 5, device=dev)
G.rqrcp(A, n, b=b, p=8, seed=0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    G.rqrcp(A, n, b=b, p=8, seed=0)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
tn = [e for e in evs if "gemm_tn_kernel" in e.name and (e.time_range.end - e.time_range.start) > 200]
nn = [e for e in evs if "gemm_nn_kernel" in e.name and (e.time_range.end - e.time_range.start) > 200]
red = [e for e in evs if "splitk_reduce" in e.name]
print("first sweeps", len(tn), "merged sweeps", len(nn), "split-K reduces", len(red),
      "reduce ms", round(sum(e.time_range.end - e.time_range.start for e in red) / 1e3, 2))
rows = []
for J, e in enumerate(tn[1:]):  # tn[0] is the sketch
    s = n - J * b
    fl = 2.0 * b * s * (s - b + (2 * b if J % 2 else b))
    us = e.time_range.end - e.time_range.start
    rows.append((J, s, us, fl / us / 1e6))
tot_us = sum(r[2] for r in rows)
ideal = sum(2.0 * b * r[1] * r[1] for r in rows) / 34.0e6
print(f"first sweeps: {tot_us / 1e3:.1f} ms; at the block-0 rate (34 TF) {ideal / 1e3:.1f} ms")
for lo, hi in [(0, 32), (32, 64), (64, 128), (128, 192), (192, 224), (224, 256)]:
    sel = [r for r in rows if lo <= r[0] < hi]
    if sel:
        print(f"  blocks {lo:3d}-{hi:3d}: {np.mean([r[3] for r in sel]):5.1f} TF avg, {sum(r[2] for r in sel) / 1e3:7.1f} ms")
rows2 = []
for q, e in enumerate(nn):
    J = 2 * q + 1
    s = n - J * b
    fl = 2.0 * 2 * b * (s + b) * (s - b)
    us = e.time_range.end - e.time_range.start
    rows2.append((J, s, us, fl / us / 1e6))
print(f"merged sweeps: {sum(r[2] for r in rows2) / 1e3:.1f} ms")
for lo, hi in [(0, 32), (32, 64), (64, 128), (128, 192), (192, 224), (224, 256)]:
    sel = [r for r in rows2 if lo <= r[0] < hi]
    if sel:
        print(f"  blocks {lo:3d}-{hi:3d}: {np.mean([r[3] for r in sel]):5.1f} TF avg, {sum(r[2] for r in sel) / 1e3:7.1f} ms")

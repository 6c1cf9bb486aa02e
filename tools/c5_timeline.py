"""torch.profiler timeline of one C5 factorization (builder tool): per-kernel
totals, the device idle time between launches, and one block pair in detail."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04447_b200 as G  # noqa: E402

dev = torch.device("cuda", 0)
n = int(os.environ.get("N", "32768"))
A = G.device_giid(n, n, 5, device=dev)
G.rqrcp(A, n, b=128, p=8, seed=0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    G.rqrcp(A, n, b=128, p=8, seed=0)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0, t1 = evs[0].time_range.start, evs[-1].time_range.end
# union of busy intervals (side streams overlap)
busy, cur_s, cur_e = 0.0, None, None
for e in evs:
    s, f = e.time_range.start, e.time_range.end
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
print(f"span {(t1 - t0) / 1e3:.1f} ms, device busy (union) {busy / 1e3:.1f} ms, idle {(t1 - t0 - busy) / 1e3:.1f} ms, "
      f"kernels {len(evs)}")
agg = {}
for e in evs:
    k = e.name.replace("(anonymous namespace)::", "").split("(")[0].split("<")[0][-48:]
    a = agg.setdefault(k, [0.0, 0])
    a[0] += e.time_range.end - e.time_range.start
    a[1] += 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:16]:
    print(f"{v[0] / 1e3:9.2f} ms {v[1]:6d}  {k}")
# one pair in the middle (blocks 100, 101): every event in order with gaps
mid = [e for e in evs if "sample_qrcp" in e.name]
blk = int(os.environ.get("BLK", "100"))  # even: the pair (blk, blk + 1), from the previous block's sample QRCP on
if len(mid) > blk + 2:
    a, b = mid[blk - 1 if blk else 0].time_range.start, mid[blk + 2].time_range.start
    prev = None
    for e in evs:
        if a <= e.time_range.start < b:
            gap = (e.time_range.start - prev) if prev is not None else 0
            print(f"{(e.time_range.start - a) / 1e3:8.3f} ms  +{gap:6.1f} us  {(e.time_range.end - e.time_range.start):8.1f} us  "
                  f"{e.name.replace('(anonymous namespace)::', '').split('(')[0].split('<')[0][-40:]}  s{e.device_resource_id if hasattr(e, 'device_resource_id') else ''}")
            prev = e.time_range.end if prev is None else max(prev, e.time_range.end)  # gap < 0: overlapped

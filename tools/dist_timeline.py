"""torch.profiler timeline of one C5 distributed RQRCP step at world size 1
(builder tool): per-kernel totals, device idle time, one mid-run block pair.

    python tools/dist_timeline.py            # NCCL
    COLL=symm python tools/dist_timeline.py  # symmetric-memory puts
"""
import os
import re
import sys

import torch
import torch.distributed as dist
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04447_b200 import distributed as D  # noqa: E402

os.environ.update({"RANK": "0", "LOCAL_RANK": "0", "WORLD_SIZE": "1", "MASTER_ADDR": "127.0.0.1",
                   "MASTER_PORT": os.environ.get("MASTER_PORT", "29533")})
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
comm = D.SymmComm(None, dev) if os.environ.get("COLL") == "symm" else D.TorchComm()
n = int(os.environ.get("N", "32768"))
b, p = 128, 8
lay = D.BlockCyclic(n, b, 1)
A0 = D.local_giid(n, n, b, 5, lay, 0, dev, rows=n + 2 * b)
ops = D.GpuOps(dev, comm)


def step():
    A = A0.clone()
    return D.rqrcp_block_cyclic(A, n, n, n, b, p, 0, comm, ops)


step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()


def nm(e):
    s = e.name.replace("(anonymous namespace)::", "")
    s = re.sub(r"<.*", "", s.split("(")[0])
    return s.replace("void ", "")[-56:]


evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0, t1 = evs[0].time_range.start, evs[-1].time_range.end
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
    k = nm(e)
    a = agg.setdefault(k, [0.0, 0])
    a[0] += e.time_range.end - e.time_range.start
    a[1] += 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:28]:
    print(f"{v[0] / 1e3:9.2f} ms {v[1]:6d}  {k}")
mid = [e for e in evs if "sample_qrcp" in e.name]
if len(mid) > 102:
    a, bnd = mid[100].time_range.start, mid[102].time_range.start
    prev = None
    for e in evs:
        if a <= e.time_range.start < bnd:
            gap = (e.time_range.start - prev) if prev is not None else 0
            print(f"{(e.time_range.start - a) / 1e3:8.3f} ms  +{gap:6.1f} us  {(e.time_range.end - e.time_range.start):8.1f} us  "
                  f"{nm(e)}")
            prev = e.time_range.end
dist.destroy_process_group()

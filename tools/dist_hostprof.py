"""cProfile of the host side of one C5 distributed RQRCP step at world size 1
(builder tool): where the per-block Python time goes."""
import cProfile
import os
import pstats
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04447_b200 import distributed as D  # noqa: E402

os.environ.update({"RANK": "0", "LOCAL_RANK": "0", "WORLD_SIZE": "1", "MASTER_ADDR": "127.0.0.1",
                   "MASTER_PORT": os.environ.get("MASTER_PORT", "29534")})
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
comm = D.TorchComm()
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
pr = cProfile.Profile()
pr.enable()
step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
dist.destroy_process_group()

"""Host -> device upload bandwidth of a C4-sized (3.2 GB) pageable array: plain
torch copy vs the pipelined pinned-staging path (_dev._h2d_pipelined)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04447_b200 import _dev  # noqa: E402

dev = torch.device("cuda", 0)
A = np.random.default_rng(0).standard_normal((20000, 20000))
d = torch.empty((20000, 20000), dtype=torch.float64, device=dev)
for name, fn in [("torch copy_ (pageable)", lambda: d.copy_(torch.from_numpy(A))),
                 ("pipelined pinned staging", lambda: _dev._h2d_pipelined(A, d))]:
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name:28s} {A.nbytes / min(ts) / 1e9:6.1f} GB/s", flush=True)
assert torch.equal(d.cpu(), torch.from_numpy(A))

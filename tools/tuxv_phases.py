"""Phase split of tuxv on C4 (20000^2, k=100, b=32): host-synchronised wall
time per stage plus libsqr kernel-class device time (builder tool)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04447_b200 as G  # noqa: E402
from paper_2008_04447_b200 import _lib, factor  # noqa: E402

dev = torch.device("cuda", 0)
n = int(os.environ.get("N", "20000"))
G1 = G.device_giid(n, 100, 41, device=dev)
G2 = G.device_giid(n, 100, 42, device=dev)
S = (G2 @ G1.T).T  # column-major (Fortran) like the reference's arrays
S /= torch.linalg.norm(S)
A = S + 1e-6 * G.device_giid(n, n, 43, device=dev)
del S
T = {}


def wrap(mod, name):
    f = getattr(mod, name)

    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = f(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
        return out
    setattr(mod, name, w)


for nm in ("trqrcp", "_qr_blocked_dev", "_q_columns_dev", "gemm_nn", "_compose_all", "_packed_blocks"):
    wrap(factor, nm)
for _ in range(2):
    G.tuxv(A, 100, b=32, p=8, seed=0)
torch.cuda.synchronize()
T.clear()
L = _lib.lib()
L.sqr_profile_enable(100000)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = G.tuxv(A, 100, b=32, p=8, seed=0)
e1.record()
torch.cuda.synchronize()
prof = _lib.profile_collect()
L.sqr_profile_enable(0)
print("total ms", round(e0.elapsed_time(e1), 2))
print("host-synced stages (ms):", {k: round(v, 2) for k, v in T.items()})
print("kernels (ms, launches):", {k: (round(v[0], 2), v[1]) for k, v in prof.items() if v[1]})

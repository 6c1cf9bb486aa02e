"""Small factorizations that reach every hand-synchronised kernel path, for
compute-sanitizer (memcheck / racecheck / synccheck):

* C1 (1000^2, b=32): cluster sample QRCP (n_t <= 16*256: DSMEM record pushes,
  hardware cluster barrier), single-launch panel, paired second sweep,
  early sample-update prep on the side stream;
* 600 x 5000 rqrcp (n_t > 4096): the grid-barrier sample QRCP with the
  deferred shared-memory updates in the barrier shadow;
* 40000 x 96 rqrcp (mr > 148*256 rows): the leaf panel kernel + WY GEMMs;
* a small C2-like TRQRCP and a TUXV (split-K GEMM, qr_blocked, result
  assembly kernels); a low-rank input (short-panel early exits, out= stream).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04447_b200 as G  # noqa: E402


def gauss(m, n, seed):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((m, n)))


def main(which):
    out = {}
    if "c1" in which:
        A = gauss(1000, 1000, 1)
        out["c1"] = G.rqrcp(A, 1000, b=32, p=8, seed=0, omega="host").perm[:8]
    if "wide" in which:
        A = gauss(600, 5000, 2)
        out["wide"] = G.rqrcp(A, 128, b=64, p=8, seed=0).perm[:8]
    if "tall" in which:
        A = gauss(40000, 96, 3)
        out["tall"] = G.rqrcp(A, 96, b=32, p=8, seed=0).perm[:8]
    if "c2" in which:
        A = gauss(1200, 1000, 4)
        out["c2"] = G.trqrcp(A, 96, b=32, p=8, seed=0).perm[:8]
    if "tuxv" in which:
        A = gauss(3000, 2500, 5)
        out["tuxv"] = G.tuxv(A, 40, b=16, p=8, seed=0).sigma_est[:4]
    if "lowrank" in which:
        rng = np.random.default_rng(6)
        A = np.asfortranarray(rng.standard_normal((200, 39)) @ rng.standard_normal((39, 180)))
        R = np.zeros((180, 180), order="F")
        out["lowrank"] = G.rqrcp(A, 180, b=16, p=8, seed=2, out=R).achieved_rank
    for k, v in out.items():
        print(k, v)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "wide", "tall", "c2", "tuxv", "lowrank"])

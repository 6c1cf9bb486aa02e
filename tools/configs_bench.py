"""Device timings of the BASELINE.json configs (builder tool, one B200).

C1 rqrcp 1000^2 b=32; C2 trqrcp 4000^2 decay k=200 b=32; C3 rqrcp
100000x2000 b=64; C4 tuxv 20000^2 rank-100 + 1e-6 noise k=100 b=32;
TRQRCP n=32768 k=3328 b=128 (SURVEY.md §8(d) extension).  Inputs are built
on the device from the reference stream; times are CUDA-event medians with
the input resident in HBM (the call includes the input copy, as the
reference's does).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04447_b200 as G  # noqa: E402
from paper_2008_04447_b200._dev import ColMajor  # noqa: E402


def timed(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), out


def decay_device(m, n, ratio, seed, dev):
    """synth_decay (synth.py:12-24) on the device: QR of stream draws, U diag(s) V^T."""
    U0 = G.device_giid(m, min(m, n), seed, 0, device=dev)
    V0 = G.device_giid(n, min(m, n), seed, m * min(m, n), device=dev)
    U, _ = torch.linalg.qr(U0)
    V, _ = torch.linalg.qr(V0)
    s = ratio ** torch.arange(min(m, n), device=dev, dtype=torch.float64)
    return (U * s) @ V.T


def main():
    dev = torch.device("cuda", 0)
    out = {}
    which = sys.argv[1:] or ["c1", "c2", "c3", "c4", "tr32k"]
    if "c1" in which:
        A = G.device_giid(1000, 1000, 1, device=dev)
        ms, pf = timed(lambda: G.rqrcp(A, 1000, b=32, p=8, seed=0), reps=5)
        out["C1_rqrcp_1000"] = {"ms": ms, "gflops_lapack": (2 * 1000 ** 3 - 2 * 1000 ** 3 / 3) / ms / 1e6,
                                "achieved": pf.achieved_rank}
    if "c2" in which:
        A = decay_device(4000, 4000, 10 ** (-10 / 4000), 2, dev)
        ms, tf = timed(lambda: G.trqrcp(A, 200, b=32, p=8, seed=0), reps=5)
        out["C2_trqrcp_4000_k200"] = {"ms": ms, "algorithmic_gflop": 8.18, "gflops": 8.18e3 / ms,
                                      "achieved": tf.achieved_rank}
    if "c3" in which:
        A = G.device_giid(100000, 2000, 3, device=dev)
        ms, pf = timed(lambda: G.rqrcp(A, 2000, b=64, p=8, seed=0), reps=3)
        g = (2.0 * 100000 * 2000 ** 2 - 2.0 * 2000 ** 3 / 3) / 1e9
        out["C3_rqrcp_100000x2000"] = {"ms": ms, "gflops_lapack": g / ms * 1e3, "achieved": pf.achieved_rank}
    if "c4" in which:
        n = 20000
        G1 = G.device_giid(n, 100, 41, device=dev)
        G2 = G.device_giid(n, 100, 42, device=dev)
        S = (G2 @ G1.T).T  # column-major (Fortran) like the reference's arrays
        S /= torch.linalg.norm(S)
        A = S + 1e-6 * G.device_giid(n, n, 43, device=dev)
        del S
        ms, res = timed(lambda: G.tuxv(A, 100, b=32, p=8, seed=0), reps=3)
        err = float(torch.linalg.norm(A - res.reconstruct_device()) / torch.linalg.norm(A))
        out["C4_tuxv_20000_k100"] = {"ms_time_to_rank_k": ms, "algorithmic_gflop": 195.3,
                                     "gflops": 195.3e3 / ms, "rel_error": err}
    if "tr32k" in which:
        A = G.device_giid(32768, 32768, 5, device=dev)
        ms, tf = timed(lambda: G.trqrcp(A, 3328, b=128, p=8, seed=0), reps=3)
        out["TRQRCP_32768_k3328"] = {"ms": ms, "algorithmic_gflop": 8187.0, "gflops": 8187e3 / ms,
                                     "achieved": tf.achieved_rank}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

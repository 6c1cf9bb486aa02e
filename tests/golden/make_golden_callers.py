"""Write tests/golden/callers.npz from the REAL reference's callers of the hot
path (sketchqr.quality.run_counters / run_quality, sketchqr.estimators) --
build container only, like make_golden.py.

    python tests/golden/make_golden_callers.py
"""
import os
import sys

import numpy as np

REF = os.environ.get("SKETCHQR_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
from sketchqr.estimators import RandomizedPivotedQR, TruncatedQLP  # noqa: E402
from sketchqr.quality import run_counters, run_quality  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def decay_matrix(m, n, ratio, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))))
    V, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))))
    s = ratio ** np.arange(min(m, n))
    return np.asfortranarray((U * s) @ V.T)


def main():
    d = {}
    X = decay_matrix(60, 40, ratio=0.8, seed=1)
    d["X"] = X
    for algo in ("qrcp", "qrcp_blocked", "ssrqrcp", "rqrcp", "rsrqrcp", "trqrcp"):
        est = RandomizedPivotedQR(rank=9, algorithm=algo, block_size=4, padding=4, random_state=5).fit(X)
        d[f"est_{algo}_sel"] = est.selected_columns_
        d[f"est_{algo}_perm"] = est.permutation_
        d[f"est_{algo}_rdiag"] = est.r_diagonal_
    q = TruncatedQLP(rank=6, block_size=4, padding=4, random_state=3)
    d["qlp_Xt"] = q.fit_transform(X)
    d["qlp_components"] = q.components_
    d["qlp_sv"] = q.singular_values_
    d["qlp_middle"] = q.middle_
    q2 = TruncatedQLP(rank=6, flip_flops=2, block_size=4, padding=4, refine_sigma=False, random_state=3)
    q2.fit(X)
    d["qlp2_sv"] = q2.singular_values_

    A = decay_matrix(48, 40, ratio=0.85, seed=2)
    d["A"] = A
    algos = ("qrcp2", "qrcp3", "qr", "ssrqrcp", "rqrcp", "rsrqrcp", "trqrcp", "tuxv")
    cnt = []
    for algo in algos:
        c = run_counters(A, algo, rank=16, block=8, pad=4, seed=7)
        cnt.append([c["achieved_rank"], c["trailing_passes"], c["blas2_volume"], c["blas3_volume"]])
    d["counters_algos"] = np.array(algos)
    d["counters"] = np.array(cnt, dtype=np.int64)
    qual = []
    qual_algos = ("qrcp2", "qrcp3", "qr", "rqrcp", "trqrcp", "tuxv", "svd")
    for algo in qual_algos:
        recs = run_quality(A, algo, rank=24, block=8, pad=4, seed=3, reps=3)
        qual.append([[r.rank, r.reps, r.err_min, r.err_median, r.err_max] for r in recs])
    d["quality_algos"] = np.array(qual_algos)
    d["quality"] = np.array(qual, dtype=np.float64)
    np.savez_compressed(os.path.join(OUT, "callers.npz"), **d)
    print("wrote callers.npz", {k: v.shape for k, v in d.items()})


if __name__ == "__main__":
    main()

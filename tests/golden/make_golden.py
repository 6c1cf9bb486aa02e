"""Write tests/golden/*.npz from the REAL reference package (build container only).

Run from the repo root:  python tests/golden/make_golden.py
It imports sketchqr from $SKETCHQR_REF (default /root/reference/pkg/src), which
exists only in the build container; the fixtures it writes are committed and
travel to the GPU box, where /root/reference does not exist.
"""
import os
import sys

import numpy as np

REF = os.environ.get("SKETCHQR_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import sketchqr  # noqa: E402
from sketchqr import rng, reference, randomized, sketch, householder, synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def gauss(m, n, seed):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((m, n)))


def pf_dict(prefix, pf, full_r=True):
    d = {f"{prefix}perm": pf.perm, f"{prefix}achieved": np.int64(pf.achieved_rank),
         f"{prefix}rdiag": pf.r_diag,
         f"{prefix}counters": np.array([pf.counters.trailing_passes, pf.counters.blas2_volume,
                                        pf.counters.blas3_volume], dtype=np.int64),
         f"{prefix}nblocks": np.int64(len(pf.blocks))}
    if full_r:
        d[f"{prefix}R"] = pf.R
        if pf.blocks:
            d[f"{prefix}tau"] = np.concatenate([b.tau for b in pf.blocks])
            d[f"{prefix}offsets"] = np.array([b.offset for b in pf.blocks], dtype=np.int64)
            d[f"{prefix}widths"] = np.array([b.width for b in pf.blocks], dtype=np.int64)
            d[f"{prefix}Ypack"] = np.hstack([b.Y for b in pf.blocks])
            d[f"{prefix}T0"] = pf.blocks[0].T
    if getattr(pf, "w_t", None) is not None and full_r:
        d[f"{prefix}w_t"] = pf.w_t
    return d


def main():
    # --- RNG: words, normals, matrices -------------------------------------
    d = {}
    d["words_seed0"] = rng._words(0, np.arange(64, dtype=np.uint64))
    d["words_big"] = rng._words(2**63 + 17, np.arange(64, dtype=np.uint64))
    d["normals_0_4096"] = rng.normals(0, 4096)
    d["normals_12345_off3"] = rng.normals(12345, 1000, offset=3)
    d["giid_40x1000_s0"] = rng.giid(40, 1000, seed=0)
    d["giid_72x333_s7_off5"] = rng.giid(72, 333, seed=7, offset=5)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **d)

    # --- Householder KATs --------------------------------------------------
    d = {}
    for i, a in enumerate([np.array([1.0, 0.0]), np.array([3.0, 4.0]), np.zeros(3),
                           np.array([-2.0, 1.0, 2.0]), gauss(17, 1, 3)[:, 0]]):
        y, tau, beta = householder.house_gen(a)
        d[f"hg{i}_a"], d[f"hg{i}_y"], d[f"hg{i}_tb"] = a, y, np.array([tau, beta])
    Y = np.tril(gauss(9, 4, 4), -1) + np.eye(9, 4)
    taus = np.array([1.2, 1.5, 0.7, 1.9])
    d["wyT_Y"], d["wyT_tau"], d["wyT_T"] = Y, taus, householder.wy_build_T(Y, taus)
    np.savez_compressed(os.path.join(OUT, "householder.npz"), **d)

    # --- deterministic QRCP oracles ------------------------------------------
    d = {}
    A = gauss(40, 30, 11)
    d["qA"] = A
    d.update(pf_dict("blas2_", reference.qrcp_blas2(A)))
    d.update(pf_dict("blocked_", reference.qrcp_blocked(A, b=8)))
    d.update(pf_dict("qrb_", reference.qr_blocked(A, b=8)))
    d.update(pf_dict("diag3_", reference.qrcp_blas2(np.diag([1.0, 2.0, 3.0]))))
    d.update(pf_dict("eye4_", reference.qrcp_blas2(np.eye(4))))
    d.update(pf_dict("diag8_", reference.qrcp_blocked(np.diag(np.arange(1.0, 9.0)), b=4)))
    np.savez_compressed(os.path.join(OUT, "qrcp.npz"), **d)

    # --- sample machinery ----------------------------------------------------
    d = {}
    B = gauss(12, 40, 5)
    st = sketch.sample_qrcp(B, 6)
    d["sB"] = B
    d["s_perm"], d["s_B_out"], d["s_achieved"] = st.local_perm, st.B, np.int64(st.achieved)
    R11 = np.triu(gauss(6, 6, 6)) + 4 * np.eye(6)
    R12 = gauss(6, 34, 7)
    d["s_R11"], d["s_R12"] = R11, R12
    d["s_next"] = sketch.sample_update(st, R11, R12)
    Bt = np.zeros((2, 3), order="F")
    Bt[:, 0] = (3.0, 4.0)
    Bt[:, 2] = (4.0, 3.0)
    Bt[:, 1] = (0.1, 0.0)
    d["tie_B"], d["tie_perm"] = Bt, sketch.sample_qrcp(Bt, 2).local_perm
    np.savez_compressed(os.path.join(OUT, "sample.npz"), **d)

    # --- randomized drivers: small cases with full outputs -------------------
    cases = {
        "r_small": ("rqrcp", gauss(200, 150, 21), dict(k=150, b=32, p=8, seed=0)),
        "r_ragged": ("rqrcp", gauss(130, 77, 22), dict(k=70, b=16, p=4, seed=3)),
        "r_tall": ("rqrcp", gauss(500, 64, 23), dict(k=64, b=16, p=8, seed=5)),
        "r_wide": ("rqrcp", gauss(60, 200, 24), dict(k=60, b=8, p=8, seed=1)),
        "r_short": ("rqrcp", gauss(30, 50, 25), dict(k=20, b=32, p=8, seed=0)),  # l >= m fallback
        "r_rankdef": ("rqrcp", np.asfortranarray(gauss(80, 10, 26) @ gauss(10, 60, 27)),
                      dict(k=40, b=8, p=8, seed=3)),
        "r_zero": ("rqrcp", np.zeros((20, 16), order="F"), dict(k=8, b=4, p=2, seed=0)),
        "r_diag64": ("rqrcp", np.asfortranarray(np.diag(np.arange(1.0, 65.0))), dict(k=64, b=8, p=8, seed=2)),
        "r_kahan": ("rqrcp", synth.synth_kahan(96), dict(k=96, b=16, p=8, seed=1)),
        "rs_small": ("rsrqrcp", gauss(120, 90, 28), dict(k=90, b=16, p=8, seed=4)),
        "ss_small": ("ssrqrcp", gauss(120, 90, 29), dict(k=24, p=8, seed=4)),
        "t_small": ("trqrcp", gauss(300, 240, 30), dict(k=64, b=16, p=8, seed=0)),
        "t_decay": ("trqrcp", synth.synth_decay(400, 300, 10 ** (-10 / 300), seed=2), dict(k=100, b=32, p=8, seed=0)),
        "t_short": ("trqrcp", gauss(20, 60, 31), dict(k=10, b=16, p=8, seed=0)),
        "t_large_k": ("trqrcp", gauss(100, 80, 32), dict(k=70, b=16, p=8, seed=0, allow_large_k=True)),
    }
    for name, (fn, A, kw) in cases.items():
        pf = getattr(randomized, fn)(A, **kw)
        d = {"A": A, "kw_keys": np.array(list(kw.keys())), "kw_vals": np.array(list(kw.values()), dtype=np.int64),
             "rel_residual": np.float64(pf.rel_residual(A))}
        d.update(pf_dict("", pf))
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)

    # --- TUXV ---------------------------------------------------------------
    for name, A, kw in [("x_small", gauss(120, 100, 40), dict(k=16, b=8, p=8, seed=0)),
                        ("x_flip2", gauss(60, 48, 41), dict(k=12, b=4, p=4, seed=5, j_max=2)),
                        ("x_refine", synth.synth_decay(80, 64, 0.7, seed=3), dict(k=10, b=8, p=8, seed=9, refine_sigma=True))]:
        res = randomized.tuxv(A, **kw)
        d = {"A": A, "kw_keys": np.array(list(kw.keys())), "kw_vals": np.array(list(kw.values()), dtype=np.int64),
             "X": res.X, "sigma_est": res.sigma_est, "achieved": np.int64(res.achieved_rank),
             "UY": res.U.Y, "UT": res.U.T, "VY": res.V.Y, "VT": res.V.T,
             "recon": res.reconstruct(),
             "counters": np.array([res.counters.trailing_passes, res.counters.blas2_volume,
                                   res.counters.blas3_volume], dtype=np.int64)}
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)

    # --- config 1 (BASELINE.md §3 inputs), summary outputs only; C2-C5: make_golden_configs.py ---
    A1 = rng.giid(1000, 1000, seed=1)
    pf = randomized.rqrcp(A1, 1000, b=32, p=8, seed=0)
    np.savez_compressed(os.path.join(OUT, "c1.npz"), **pf_dict("", pf, full_r=False),
                        rel_residual=np.float64(pf.rel_residual(A1)))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()

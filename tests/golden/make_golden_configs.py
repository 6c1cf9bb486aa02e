"""Reference outputs at BASELINE.json's full configs C2, C3, C4 and C5, written by
the REAL reference package (build container only; /root/reference does not
exist on the GPU box).

    python tests/golden/make_golden_configs.py c2 c3 c4   # minutes
    python tests/golden/make_golden_configs.py c5         # ~2 h, ~45 GB RAM

Each fixture holds what the GPU parity tests compare (perm, |R| diagonal,
counters, achieved rank; for C4 also X, sigma_est and the truncation error)
plus the sha256 of the input bytes (config_inputs.column_digest), the
reference wall time and the host it ran on.  C2's fixture is written by
this script too (c2.npz; make_golden.py writes the small cases and C1).
"""
import json
import os
import platform
import sys
import time

import numpy as np

REF = os.environ.get("SKETCHQR_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
from sketchqr import randomized, rng, synth  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import config_inputs as CI  # noqa: E402


def host_info():
    info = {"cpus": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "machine": platform.machine(), "numpy": np.__version__}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "architecture")}
                        for d in threadpool_info()]
    except Exception:  # pragma: no cover
        pass
    return json.dumps(info)


def counters(c):
    return np.array([c.trailing_passes, c.blas2_volume, c.blas3_volume], dtype=np.int64)


def run_c2():
    """C2: TRQRCP k=200 of synth_decay(4000, 4000, 10**(-10/4000), seed=2)."""
    A = synth.synth_decay(4000, 4000, ratio=10 ** (-10 / 4000), seed=2)
    digest = CI.column_digest(A)
    t0 = time.perf_counter()
    tf = randomized.trqrcp(A, 200, b=32, p=8, seed=0)
    t = time.perf_counter() - t0
    np.savez_compressed(os.path.join(HERE, "c2.npz"), perm=tf.perm, rdiag=tf.r_diag,
                        achieved=np.int64(tf.achieved_rank), counters=counters(tf.counters),
                        nblocks=np.int64(len(tf.blocks)), R_top=tf.R[:, :200],
                        rel_residual=np.float64(tf.rel_residual(A, 200)), w_t_head=tf.w_t[:, 200:456],
                        sha256=np.array(digest), seconds=np.float64(t), host=np.array(host_info()))
    print(f"c2: {t:.2f} s rel_err {tf.rel_residual(A, 200):.10e} sha {digest[:16]}", flush=True)


def run_c3():
    A = CI.c3_matrix(rng.normals)
    digest = CI.column_digest(A)
    t0 = time.perf_counter()
    pf = randomized.rqrcp(A, 2000, b=64, p=8, seed=0)
    t = time.perf_counter() - t0
    np.savez_compressed(os.path.join(HERE, "c3.npz"), perm=pf.perm, rdiag=pf.r_diag,
                        achieved=np.int64(pf.achieved_rank), counters=counters(pf.counters),
                        nblocks=np.int64(len(pf.blocks)), R_head=pf.R[:64, :256],
                        sha256=np.array(digest), seconds=np.float64(t), host=np.array(host_info()))
    print(f"c3: {t:.1f} s achieved {pf.achieved_rank} sha {digest[:16]}", flush=True)


def run_c4():
    A = CI.c4_matrix(rng.normals)
    digest = CI.column_digest(A)
    t0 = time.perf_counter()
    res = randomized.tuxv(A, 100, b=32, p=8, seed=0)
    t = time.perf_counter() - t0
    t0 = time.perf_counter()
    tf = randomized.trqrcp(A, 100, b=32, p=8, seed=0)
    t_tr = time.perf_counter() - t0
    # truncation error ||A - U X V^T||_F / ||A||_F, formed block-wise
    Uk = res.u_columns()
    Vk = res.v_columns()
    UX = Uk @ res.X
    err2 = 0.0
    for j0 in range(0, A.shape[1], 2000):
        D = A[:, j0:j0 + 2000] - UX @ Vk[j0:j0 + 2000].T
        err2 += float(np.einsum("ij,ij->", D, D))
    rel_err = np.sqrt(err2) / np.linalg.norm(A)
    np.savez_compressed(os.path.join(HERE, "c4.npz"), X=res.X, sigma_est=res.sigma_est,
                        achieved=np.int64(res.achieved_rank), counters=counters(res.counters),
                        rel_error=np.float64(rel_err), t_perm=tf.perm, t_rdiag=tf.r_diag,
                        t_counters=counters(tf.counters), Vk_head=Vk[:64], Uk_head=Uk[:64],
                        sha256=np.array(digest), seconds=np.float64(t), trqrcp_seconds=np.float64(t_tr),
                        host=np.array(host_info()))
    print(f"c4: tuxv {t:.1f} s trqrcp {t_tr:.1f} s rel_err {rel_err:.6e} sha {digest[:16]}", flush=True)


def run_c5():
    t0 = time.perf_counter()
    A = CI.c5_matrix(rng.normals)
    tgen = time.perf_counter() - t0
    digest = CI.column_digest(A)
    print(f"c5: A generated in {tgen:.1f} s sha {digest[:16]}", flush=True)
    t0 = time.perf_counter()
    pf = randomized.rqrcp(A, 32768, b=128, p=8, seed=0)
    t = time.perf_counter() - t0
    rdiag = pf.r_diag
    np.savez_compressed(os.path.join(HERE, "c5.npz"), perm=pf.perm, rdiag=rdiag,
                        achieved=np.int64(pf.achieved_rank), counters=counters(pf.counters),
                        nblocks=np.int64(len(pf.blocks)), R_head=pf.R[:128, :512],
                        sha256=np.array(digest), seconds=np.float64(t), host=np.array(host_info()))
    print(f"c5: {t:.1f} s achieved {pf.achieved_rank} counters {counters(pf.counters)}", flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c2", "c3", "c4"]:
        {"c2": run_c2, "c3": run_c3, "c4": run_c4, "c5": run_c5}[name]()

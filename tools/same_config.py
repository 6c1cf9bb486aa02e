"""Same-config CPU-vs-GPU timings of BASELINE.json configs C1-C4 on ONE box
(SURVEY.md §8(d) "CPU baseline timing"): the identical host-generated inputs
(tests/golden/config_inputs.py, the reference's counter-based stream) go to

* the CPU oracle port (oracle/port.py: the reference's algorithm restated in
  NumPy -> OpenBLAS, all host threads; /root/reference cannot travel to the
  GPU box, and the port is pinned bit-for-bit to it by tests/test_oracle.py),
  timed with time.perf_counter around the call only (C1/C2 median of 3,
  C3/C4 one run);
* the GPU package's default call (Omega drawn on the device), end to end
  from the host array (H2D, factorization, the result's host arrays: R +
  perm / w_t / X, sigma, U.Y, V.Y) and device-only with the input resident in
  HBM (CUDA events, median of 3).

    python tools/same_config.py [c1 c2 c3 c4] > profiles/configs_r02.json
"""
import json
import os
import platform
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import config_inputs as CI  # noqa: E402
import paper_2008_04447_b200 as G  # noqa: E402
from oracle import port as O  # noqa: E402


def host_info():
    info = {"cpus": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "machine": platform.machine()}
    try:
        with open("/proc/cpuinfo") as f:
            info["model"] = next(ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name"))
    except (OSError, StopIteration):
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads")} for d in threadpool_info()]
    except Exception:
        pass
    return info


def wall(fn, reps):
    ts, out = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), out


def dev_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def e2e(fn, fetch, reps=3):
    fetch(fn())
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fetch(fn())
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def lapack(m, n):
    return (2.0 * m * n * n - 2.0 * n ** 3 / 3) / 1e9


CONFIGS = {
    "c1": dict(inp=lambda: O.gauss_matrix(1000, 1000, 1), call="rqrcp", args=(1000,), kw=dict(b=32, p=8, seed=0),
               gflop=lapack(1000, 1000), conv="LAPACK", reps=3),
    "c2": dict(inp=lambda: O.synth_decay(4000, 4000, ratio=10 ** (-10 / 4000), seed=2), call="trqrcp", args=(200,),
               kw=dict(b=32, p=8, seed=0), gflop=8.18, conv="algorithmic", reps=3),
    "c3": dict(inp=lambda: CI.c3_matrix(O.gauss_stream), call="rqrcp", args=(2000,), kw=dict(b=64, p=8, seed=0),
               gflop=lapack(100000, 2000), conv="LAPACK", reps=1),
    "c4": dict(inp=lambda: CI.c4_matrix(O.gauss_stream), call="tuxv", args=(100,), kw=dict(b=32, p=8, seed=0),
               gflop=195.3, conv="algorithmic", reps=1),
}


def fetch(res):
    """The result's host arrays, as the reference returns them."""
    if hasattr(res, "sigma_est"):
        return res.X, res.sigma_est, res.U.Y, res.V.Y
    out = [res.R, res.perm]
    if hasattr(res, "w_t"):
        out.append(res.w_t)
    return out


def main():
    which = sys.argv[1:] or list(CONFIGS)
    dev = torch.device("cuda", 0)
    out = {"host": host_info(), "configs": {}}
    for name in which:
        c = CONFIGS[name]
        A = c["inp"]()
        cpu_s, _ = wall(lambda: getattr(O, c["call"])(A, *c["args"], **c["kw"]), c["reps"])
        gfn = getattr(G, c["call"])
        # the drop-in default call (Omega drawn on the device); parity of both
        # Omega modes against the reference: tests/test_gpu_configs.py
        t_e2e = e2e(lambda: gfn(A, *c["args"], **c["kw"]), fetch)
        Ad = torch.from_numpy(A).to(dev)
        ms = dev_ms(lambda: gfn(Ad, *c["args"], **c["kw"]))
        out["configs"][name] = {
            "call": f"{c['call']}{c['args']} {c['kw']}", "shape": list(A.shape), "gflop": c["gflop"],
            "flop_convention": c["conv"],
            "cpu_oracle_port_s": cpu_s, "cpu_gflops": c["gflop"] / cpu_s,
            "gpu_e2e_s": t_e2e, "gpu_e2e_gflops": c["gflop"] / t_e2e,
            "gpu_device_ms": ms, "gpu_device_gflops": c["gflop"] / ms * 1e3,
            "speedup_e2e": cpu_s / t_e2e, "speedup_device": cpu_s / (ms / 1e3),
            "cpu_reps": c["reps"]}
        print(name, json.dumps(out["configs"][name]), file=sys.stderr, flush=True)
        del A, Ad
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

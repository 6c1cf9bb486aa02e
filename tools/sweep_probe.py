"""First / second sweep GEMM throughput over the C5 block sizes (builder tool):
gemm_tn(128, s, s) with the Y prefix off, gemm_nn(s, s, 256) for s = n - i0."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04447_b200 import _lib  # noqa: E402
from paper_2008_04447_b200._dev import stream_handle  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
ws = torch.zeros(400 << 20, dtype=torch.uint8, device=dev)
st = stream_handle()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for s in [int(x) for x in (sys.argv[1:] or ["32768", "24576", "16384", "12288", "8192", "6144", "4096", "2048", "1024"])]:
    C = torch.randn((s, s), dtype=torch.float64, device=dev, generator=g)
    Y = torch.randn((256, s), dtype=torch.float64, device=dev, generator=g) * 1e-3
    W = torch.randn((s, 256), dtype=torch.float64, device=dev, generator=g) * 1e-3
    D = torch.empty((s, 128), dtype=torch.float64, device=dev)
    t_tn = timed(lambda: _lib.check(L.sqr_gemm_tn(128, s, s, 1.0, Y.data_ptr(), s, C.data_ptr(), s, 0.0, None, 0,
                                                 D.data_ptr(), 128, ws.data_ptr(), ws.numel(), st)))
    t_nn = timed(lambda: _lib.check(L.sqr_gemm_nn(s, s, 256, 1.0, Y.data_ptr(), s, W.data_ptr(), 256, 1.0, C.data_ptr(),
                                                 s, C.data_ptr(), s, st)))
    f_tn, f_nn = 2.0 * 128 * s * s, 2.0 * 256 * s * s
    print(f"s={s:6d}  tn {t_tn * 1e3:9.1f} us {f_tn / t_tn / 1e9:6.2f} TF   nn(K=256) {t_nn * 1e3:9.1f} us "
          f"{f_nn / t_nn / 1e9:6.2f} TF", flush=True)
    del C, Y, W, D
    torch.cuda.empty_cache()

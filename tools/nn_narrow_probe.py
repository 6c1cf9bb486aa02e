"""Short-M gemm_nn (M = 128, K = 128) over N: 64- vs 32-wide N tiles (builder
tool; run twice, with and without SQR_NO_NARROW_NN=1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04447_b200 import _lib  # noqa: E402
from paper_2008_04447_b200._dev import stream_handle  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
s = stream_handle()
M = K = 128
for N in [int(x) for x in (sys.argv[1:] or ["8000", "12000", "16000", "19500", "20000", "24000", "28000", "32640"])]:
    X = torch.randn((K, M), dtype=torch.float64, device=dev, generator=g)
    Y = torch.randn((N, K), dtype=torch.float64, device=dev, generator=g)
    E = torch.randn((N, M), dtype=torch.float64, device=dev, generator=g)

    def run():
        _lib.check(L.sqr_gemm_nn(M, N, K, -1.0, X.data_ptr(), M, Y.data_ptr(), K, 1.0, E.data_ptr(), M, E.data_ptr(),
                                 M, s))
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(20):
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"N={N:6d}  {best * 1e3:7.1f} us  {2.0 * M * N * K / best / 1e9:6.2f} TF", flush=True)

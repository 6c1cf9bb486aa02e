"""gemm_nn throughput vs the update rank K on the C5 trailing shape (builder
tool: how much a merged multi-block second sweep would gain)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04447_b200 import _lib  # noqa: E402
from paper_2008_04447_b200._dev import stream_handle  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda", 0)
m, n = 32768, 32640
g = torch.Generator(device=dev).manual_seed(0)
C = torch.randn((n, m), dtype=torch.float64, device=dev, generator=g)
s = stream_handle()
for K in [int(x) for x in (sys.argv[1:] or ["128", "256", "384", "512"])]:
    Y = torch.randn((K, m), dtype=torch.float64, device=dev, generator=g) * 1e-3
    W = torch.randn((n, K), dtype=torch.float64, device=dev, generator=g) * 1e-3

    def run():
        beta = float(os.environ.get("NN_BETA", "1"))
        _lib.check(L.sqr_gemm_nn(m, n, K, 1.0, Y.data_ptr(), m, W.data_ptr(), K, beta, C.data_ptr(), m,
                                 C.data_ptr(), m, s))
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"K={K:4d}  {best:8.3f} ms  {2.0 * m * n * K / best / 1e9:6.2f} TFLOP/s", flush=True)

"""cuBLAS DGEMM (torch.matmul, fp64) vs libsqr's DMMA GEMMs on the C5 trailing-
update shapes: the first sweep Y^T C (M = b = 128, long K) and the merged
second sweep C += [Y_P|Y_J][W_P;W_J] (K = 2b = 256), at block 0 and at a
mid-run block.  CUDA-event medians of 5; fp64 peak 37.0 TFLOP/s."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04447_b200 import _lib  # noqa: E402
from paper_2008_04447_b200._dev import stream_handle  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda", 0)
ws = torch.zeros(400 << 20, dtype=torch.uint8, device=dev)


def t(fn, reps=5):
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


for mr in (32768, 16384):
    nt = mr - 128
    g = torch.Generator(device=dev).manual_seed(0)
    C = torch.randn((nt, mr), dtype=torch.float64, device=dev, generator=g)       # column-major mr x nt
    Y = torch.randn((256, mr), dtype=torch.float64, device=dev, generator=g)      # column-major mr x 256
    W = torch.randn((nt, 256), dtype=torch.float64, device=dev, generator=g)      # column-major 256 x nt
    D = torch.empty((nt, 128), dtype=torch.float64, device=dev)
    s = stream_handle()
    fl_tn = 2.0 * 128 * mr * nt
    ms = t(lambda: _lib.check(L.sqr_gemm_tn(128, nt, mr, 1.0, Y.data_ptr(), mr, C.data_ptr(), mr, 0.0, None, 0,
                                            D.data_ptr(), 128, ws.data_ptr(), ws.numel(), s)))
    Yt = Y[:128]            # (128, mr): Y^T as a row-major view
    ms_cb = t(lambda: torch.matmul(Yt, C.T))                                    # (128 x mr)(mr x nt)
    print(f"first sweep mr={mr}: libsqr {fl_tn / ms / 1e9:.1f} TF  cuBLAS {fl_tn / ms_cb / 1e9:.1f} TF", flush=True)
    fl_nn = 2.0 * mr * nt * 256
    Cm = C.clone()
    ms = t(lambda: _lib.check(L.sqr_gemm_nn(mr, nt, 256, 1.0, Y.data_ptr(), mr, W.data_ptr(), 256, 1.0,
                                            Cm.data_ptr(), mr, Cm.data_ptr(), mr, s)))
    Ym, Wm, Cc = Y.T, W.T, C.T   # (mr, 256), (256, nt), (mr, nt) column-major views
    ms_cb = t(lambda: Cc.addmm_(Ym, Wm))
    print(f"merged second sweep mr={mr}: libsqr {fl_nn / ms / 1e9:.1f} TF  cuBLAS {fl_nn / ms_cb / 1e9:.1f} TF",
          flush=True)
    del C, Cm, Y, W, D
    torch.cuda.empty_cache()

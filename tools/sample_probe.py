"""Time sqr_sample_qrcp (C5 sample shape ell = 136, bb = 128) at several sample
widths: the pivot-epoch kernel (default) against the per-pivot-barrier kernel
(default; SQR_EPOCH_SAMPLE=1 selects the epoch kernel, read per call).  With SQR_TRACE=1 also prints the
epoch kernel's leader timeline (epochs, per-step time) from the debug trace.

    python tools/sample_probe.py [nt ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04447_b200 import _lib  # noqa: E402
from paper_2008_04447_b200._dev import ColMajor, status_new, status_read, stream_handle  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda", 0)
ell, bb = 136, 128
NTS = [int(a) for a in sys.argv[1:]] or [32768, 24576, 16384, 8192, 4096, 2048, 1024, 256]
nmax = max(NTS)
g = torch.Generator(device=dev).manual_seed(0)
B = ColMajor(torch.randn((nmax, ell), dtype=torch.float64, device=dev, generator=g), ell, nmax, ell)
Bf = ColMajor.empty(ell, nmax, dev)
lperm = torch.empty(nmax, dtype=torch.int64, device=dev)
moves = torch.empty(4 * bb + 8, dtype=torch.int32, device=dev)
taus = torch.zeros(bb, dtype=torch.float64, device=dev)
st = status_new(dev)
s = stream_handle()


def run(nt, epoch):
    if epoch:
        os.environ["SQR_EPOCH_SAMPLE"] = "1"
    else:
        os.environ.pop("SQR_EPOCH_SAMPLE", None)
    st.zero_()
    _lib.check(L.sqr_sample_qrcp(B.ptr, B.ld, ell, nt, bb, Bf.ptr, Bf.ld, lperm.data_ptr(), moves.data_ptr(),
                                 taus.data_ptr(), 1, st.data_ptr(), s))


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
    return best * 1e3


for nt in NTS:
    t_new = timed(lambda: run(nt, True))
    p_new = lperm[:bb].clone()
    t_old = timed(lambda: run(nt, False))
    same = bool(torch.equal(p_new, lperm[:bb]))
    print(f"nt={nt:6d}  epoch {t_new:8.1f} us  per-pivot-barrier {t_old:8.1f} us  x{t_old / t_new:5.2f}  "
          f"same pivots: {same}", flush=True)
    if os.environ.get("SQR_TRACE"):
        tr = torch.zeros(8 * 256, dtype=torch.int64, device=dev)
        L.sqr_debug_trace(tr.data_ptr())
        run(nt, True)
        torch.cuda.synchronize()
        L.sqr_debug_trace(None)
        t = tr.cpu().numpy().astype(np.float64)
        st8 = t[:8 * bb].reshape(bb, 8)
        ep = t[1024:1088]
        ep = ep[ep > 0]
        t0 = ep[0]
        print("   epochs:", ep.size, "starts (us):", ((ep - t0) / 1e3).round(1).tolist())
        ok = st8[:, 0] > 0
        S = st8[ok]
        names = ["argmax(lbar1)", "reflector", "apply(w0)", "publish(from lbar2)", "apply(w6)"]
        pairs = [(0, 1), (1, 4), (4, 5), (4, 6), (4, 7)]
        for nm, (i, k) in zip(names, pairs):
            v = (S[:, k] - S[:, i]) / 1e3
            print("   %-20s median %.2f  mean %.2f  max %.2f us" % (nm, np.median(v), v.mean(), v.max()))
        c_ = np.diff(S[:, 0]) / 1e3
        print("   %-20s median %.2f  mean %.2f  max %.2f us" % ("step->step", np.median(c_), c_.mean(), c_.max()))
        k0 = t[1102]
        print("   leader entry -> epoch0 %.1f, worker0 publish(0) done %.1f, leader final post %.1f, "
              "worker0 loop exit %.1f, worker0 exit %.1f us (worker0 entry %.1f)" % tuple(
                  (t[i] - k0) / 1e3 for i in (1024, 1104, 1103, 1105, 1101, 1100)))
        print("   worker0: loaded %.1f, norms %.1f, sorted %.1f, written %.1f us" % tuple((t[i] - k0) / 1e3 for i in (1110, 1111, 1112, 1113)))
        sel = t[1130:1194][:ep.size]
        fs = [S[S[:, 0] > e, 0].min() if (S[:, 0] > e).any() else np.nan for e in ep]
        print("   epoch: selection us", ((sel - ep) / 1e3).round(1).tolist())
        print("   epoch: load us     ", ((np.array(fs) - sel) / 1e3).round(1).tolist())
        ck = t[1200:2000].reshape(100, 8)[:, :4]
        print("   cycles (median): argmax %d, x+partial %d, scalar+y %d, apply %d" % tuple(np.median(ck, axis=0)))
        print("   cycles (mean):   argmax %d, x+partial %d, scalar+y %d, apply %d" % tuple(np.mean(ck, axis=0)))
        print("   first step at %.1f us after epoch 0, last step start at %.1f us, kernel %.1f us" % (
            (S[0, 0] - t0) / 1e3, (S[:, 0].max() - t0) / 1e3, t_new))
os.environ.pop("SQR_EPOCH_SAMPLE", None)
print("status", status_read(st))

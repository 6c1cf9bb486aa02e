"""Per-column cycle split of panel_block_kernel (CTA 0, thread 0) on a 32768 x 128
panel.  Needs a build with the probe compiled in:
    python -m paper_2008_04447_b200.build -DSQR_PANEL_CK --name=libsqr_ck.so
    SQR_LIB=libsqr_ck.so python tools/panel_cycles.py
"""
import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2008_04447_b200 import _lib
from paper_2008_04447_b200._dev import ColMajor, status_new, stream_handle
L = _lib.lib(); dev = torch.device("cuda", 0)
m, b = 32768, 128
P0 = torch.randn((b, m), dtype=torch.float64, device=dev)
P = ColMajor(P0.clone(), m, b, m); Y = ColMajor.empty(m, b, dev)
taus = torch.zeros(b, dtype=torch.float64, device=dev); st = status_new(dev)
ws = torch.zeros(int(L.sqr_block_workspace(m, 0, b)), dtype=torch.uint8, device=dev)
def run():
    P.t.copy_(P0); st.zero_()
    _lib.check(L.sqr_panel_factor(P.ptr, P.ld, m, b, Y.ptr, Y.ld, taus.data_ptr(), 1, st.data_ptr(), ws.data_ptr(), ws.numel(), stream_handle()))
run(); torch.cuda.synchronize()
tr = torch.zeros(2048, dtype=torch.int64, device=dev)
L.sqr_debug_trace(tr.data_ptr()); run(); torch.cuda.synchronize(); L.sqr_debug_trace(None)
c = tr.cpu().numpy()[1200:2000].reshape(100, 8)[:, :6].astype(float)
names = ["products+butterfly", "warp-sum+store", "grid barrier", "partials load+reduce", "scalars+wv", "update+shift"]
print("median cycles per column:", dict(zip(names, np.median(c[:96], axis=0).astype(int))))
print("mean:", dict(zip(names, np.mean(c[:96], axis=0).astype(int))), "sum median", int(np.median(c[:96], axis=0).sum()))

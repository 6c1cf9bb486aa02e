"""Panel kernel probe: time sqr_panel_factor (panel_block_kernel) on random
panels (--trace: the kernel's %globaltimer phase stamps of each leaf
boundary).  Used for the CholQR2-leaf experiment recorded in DESIGN.md §3
(status aux[0] / aux[1] were its leaf / fallback counters).

    python tools/panel_probe.py [--shape 32768x128] [--trace] [--save out.npz]
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
out = {}
shapes = [(32768, 128), (16384, 128), (4096, 128), (30000, 64), (1000, 32)]
if "--shape" in sys.argv:
    mr_s, w_s = sys.argv[sys.argv.index("--shape") + 1].split("x")
    shapes = [(int(mr_s), int(w_s))]
for mr, w in shapes:
    rng = np.random.default_rng(mr + w)
    P0 = torch.from_numpy(np.ascontiguousarray(rng.standard_normal((w, mr)))).to(dev)   # (w, mr): column-major
    Y = ColMajor.empty(mr, w, dev)
    taus = torch.zeros(w, dtype=torch.float64, device=dev)
    ws = torch.zeros(int(L.sqr_block_workspace(mr, 0, w)) + 4096, dtype=torch.uint8, device=dev)
    ts = []
    for rep in range(12):
        P = P0.clone()
        st = status_new(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.sqr_panel_factor(P.data_ptr(), mr, mr, w, Y.ptr, Y.ld, taus.data_ptr(), 1, st.data_ptr(),
                                      ws.data_ptr(), ws.numel(), stream_handle()))
        e1.record()
        e1.synchronize()
        if rep >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    s = status_read(st)
    if "--trace" in sys.argv:
        tr = torch.zeros(1024, dtype=torch.int64, device=dev)
        L.sqr_debug_trace(tr.data_ptr())
        P = P0.clone()
        st = status_new(dev)
        _lib.check(L.sqr_panel_factor(P.data_ptr(), mr, mr, w, Y.ptr, Y.ld, taus.data_ptr(), 1, st.data_ptr(),
                                      ws.data_ptr(), ws.numel(), stream_handle()))
        torch.cuda.synchronize()
        L.sqr_debug_trace(None)
        t = tr.cpu().numpy().astype(np.int64)
        c1 = [int(t[8 * c + 1]) for c in range(min(w, 40))]
        c2 = [int(t[8 * c + 2]) for c in range(min(w, 40))]
        if c1[0]:
            steps = [c1[i + 1] - c1[i] for i in range(min(w, 40) - 1) if c1[i + 1] and c1[i]]
            bars = [c2[i] - c1[i] for i in range(min(w, 40)) if c2[i] and c1[i]]
            print(f"  per-column step (ns): median {int(np.median(steps))}  barrier wait of CTA 0 median "
                  f"{int(np.median(bars))}  (columns 0..{min(w, 40) - 1})", flush=True)
        for li in range(w // 32):
            bd = t[8 * (40 + li):8 * (40 + li) + 8]
            if bd[0]:
                print(f"  leaf {li} boundary stamps (ns from leaf start): " +
                      " ".join(str(int(x - bd[7])) if x else "-" for x in bd), flush=True)
    key = f"{mr}x{w}"
    out[key] = P.cpu().numpy()
    out[key + "_tau"] = taus.cpu().numpy()
    print(f"{key}: {np.median(ts):8.1f} us  cholqr leaves {s['aux'][0]:.0f} fallbacks {s['aux'][1]:.0f} "
          f"bhat {int(s['bhat'])}", flush=True)
if "--save" in sys.argv:
    np.savez(sys.argv[sys.argv.index("--save") + 1], **out)

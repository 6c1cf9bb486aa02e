"""RQRCP / RSRQRCP / TRQRCP for block sizes beyond the fused driver's limits
(b > 128 or b + p > 144).

The reference accepts any b >= 1, p >= 0 (validation.py:75-82).  libsqr's
one-launch drivers (sqr_rqrcp / sqr_trqrcp) keep a 128-wide panel and a
<= 144-row sample in registers / shared memory; wider blocks run here, one
block per loop iteration with a host synchronisation per block, on the same
kernels:

* the sample QRCP of the l x n_t sample (the shared-memory / L2-spill
  cooperative kernel takes any l);
* the block's panel (randomized.py:107-130) as sub-panels of <= 128 columns:
  each sub-panel is factored by the panel kernel and its reflectors are then
  applied to the panel columns right of it -- the reference's right-looking
  loop, reflector by reflector, regrouped; a zero column inside sub-panel s
  stops the panel exactly where the reference's loop breaks;
* the block reflection Q^T C of the trailing matrix (randomized.py:203-207)
  as the sub-blocks' reflections in order, Q^T = Q_s^T ... Q_1^T;
* the sample update (sketch.py:132-149) with a general triangular solve
  (sqr_trsm_right_upper) and a DMMA GEMM.

Same pivots, early exits and counters as the reference; only the grouping of
the floating-point work differs (rounding-level).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._dev import ColMajor, ptr, status_new, status_read, stream_handle
from .counters import rqrcp_counters, trqrcp_counters

_DIAG_FLOOR = 2.0 ** -52
_SUB = 128          # widest panel the panel kernel / block update take


def _ws(nbytes, dev):
    from ._dev import Workspace
    return Workspace.lease(nbytes, dev)


class _Loop:
    """Per-factorization buffers and the per-block kernels."""

    def __init__(self, M: ColMajor, b: int, ell: int):
        self.M, self.b, self.ell = M, b, ell
        self.m, self.n = M.m, M.n
        self.dev = M.t.device
        self.L = _lib.lib()
        n, dev = self.n, self.dev
        self.Bf = ColMajor.empty(ell, n, dev)
        self.lperm = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        self.moves = torch.empty(4 * b + 8, dtype=torch.int32, device=dev)
        self.staus = torch.zeros(b, dtype=torch.float64, device=dev)
        self.st = status_new(dev)
        self.sws = torch.zeros(int(self.L.sqr_sample_qrcp_workspace(ell, n)) + 4096, dtype=torch.uint8, device=dev)
        self.floor = None

    def chk(self, rc, what):
        _lib.check(rc, what)

    def sample_qrcp(self, B: ColMajor, nt: int, bb: int):
        """(stop, reason, sample_achieved); the first call fixes the sample floor."""
        self.st.zero_()
        first = self.floor is None
        if not first:
            self.st[32:40].view(torch.float64).fill_(self.floor)
        self.chk(self.L.sqr_sample_qrcp_ws(B.ptr, B.ld, self.ell, nt, bb, self.Bf.ptr, self.Bf.ld, ptr(self.lperm),
                                           ptr(self.moves), ptr(self.staus), 1 if first else 0, ptr(self.st),
                                           ptr(self.sws), self.sws.numel(), stream_handle()), "sample_qrcp")
        s = status_read(self.st)
        if first:
            self.floor = float(s["floor_sq"])
        return bool(s["stop"]), int(s["reason"]), int(s["sample_achieved"])

    def apply_moves(self, X: ColMajor, rows: int, col0: int, perm, bb: int):
        self.chk(self.L.sqr_apply_moves(X.ptr, X.ld, rows, col0, ptr(perm) if perm is not None else None,
                                        ptr(self.moves), ptr(self.st), 2 * bb, stream_handle()), "apply_moves")

    def block_update(self, C_ptr: int, ldc: int, mr: int, ncols: int, Y: ColMajor, bh: int, taus_ptr: int):
        """C := (I - Y T Y^T)^T C for a sub-block of bh <= 128 reflectors."""
        if ncols <= 0 or bh <= 0:
            return
        T = torch.empty(bh * bh, dtype=torch.float64, device=self.dev)
        with _ws(self.L.sqr_block_workspace(mr, ncols, bh), self.dev) as ws:
            self.chk(self.L.sqr_apply_block_update(C_ptr, ldc, mr, ncols, bh, Y.ptr, Y.ld, taus_ptr, ptr(T), bh,
                                                   ptr(ws), ws.numel(), stream_handle()), "block_update")

    def panel(self, P: ColMajor, r0: int, c0: int, sa: int, taus: torch.Tensor, t0: int):
        """Panel QR of the sa columns at P[r0:, c0:c0+sa] in sub-panels; returns
        (bhat, [(offset, width, Y)]) with Y explicit, rows from r0 + offset."""
        subs = []
        bhat = 0
        for s0 in range(0, sa, _SUB):
            w = min(_SUB, sa - s0)
            mr = P.m - r0 - s0
            Y = ColMajor.empty(mr, w, self.dev)
            pst = status_new(self.dev)
            base = P.col_ptr(r0 + s0, c0 + s0)
            tp = taus.data_ptr() + 8 * (t0 + s0)
            with _ws(self.L.sqr_block_workspace(mr, 0, w), self.dev) as ws:
                self.chk(self.L.sqr_panel_factor(base, P.ld, mr, w, Y.ptr, Y.ld, tp, 1, ptr(pst), ptr(ws), ws.numel(),
                                                 stream_handle()), "panel")
            s = status_read(pst)
            bh = 0 if int(s["stop"]) else int(s["bhat"])
            if bh:
                subs.append((s0, bh, Y))
                # the reference applies each reflector to every later panel column
                self.block_update(P.col_ptr(r0 + s0, c0 + s0 + w), P.ld, mr, sa - s0 - w, Y, bh, tp)
            bhat = s0 + bh
            if bh < w:
                break
        return bhat, subs

    def sample_update(self, nt: int, bb: int, R_ptr: int, ldr: int) -> ColMajor:
        """B_next = [S12 - S11 R11^{-1} R12 ; S22] (sketch.py:132-149); R = [R11 | R12]."""
        ell, dev = self.ell, self.dev
        nn = nt - bb
        Mm = ColMajor.empty(bb, bb, dev)
        self.chk(self.L.sqr_trsm_right_upper(self.Bf.ptr, self.Bf.ld, bb, bb, R_ptr, ldr, Mm.ptr, Mm.ld, 1,
                                             stream_handle()), "trsm")
        Bn = ColMajor.empty(ell, nn, dev)
        S12 = self.Bf.col_ptr(0, bb)
        self.chk(self.L.sqr_gemm_nn(bb, nn, bb, -1.0, Mm.ptr, Mm.ld, R_ptr + 8 * bb * ldr, ldr, 1.0, S12,
                                    self.Bf.ld, Bn.ptr, Bn.ld, stream_handle()), "sample_update")
        if ell > bb:
            Bn.view()[bb:, :] = self.Bf.view()[bb:, bb:nt]
        return Bn


def _r11_ok(M: ColMajor, i0: int, bh: int) -> bool:
    """_diag_ok (randomized.py:133-135) on R11 = M[i0:i0+bh, i0:i0+bh]."""
    d = torch.diagonal(M.view()[i0:i0 + bh, i0:i0 + bh]).abs().cpu().numpy()
    return d.size > 0 and d.min() > _DIAG_FLOOR * d[0]


def _sketch(M: ColMajor, OmT: ColMajor | None, ell: int, seed: int, offset: int, r0: int = 0) -> ColMajor:
    """B = Omega A[r0:, r0:] with Omega = stream draw at `offset` (rng.py:85-93) or OmT given."""
    from .factor import gemm_tn
    m, n = M.m - r0, M.n - r0
    if OmT is None:
        OmT = ColMajor.empty(m, ell, M.t.device)
        _lib.check(_lib.lib().sqr_gaussian(OmT.ptr, OmT.ld, ell, m, seed & ((1 << 64) - 1), offset, 1,
                                           stream_handle()), "sqr_gaussian")
    return gemm_tn(OmT, ColMajor(M.t[r0:, r0:], m, n, M.ld))


def rqrcp_wide(M: ColMajor, k: int, b: int, p: int, seed: int, resample: bool, OmT):
    """randomized.py:166-224 for any b (see module docstring); M is factored in place."""
    from .factor import PivotedFactorization, _packed_blocks, _upper_rows
    m, n = M.m, M.n
    ell = b + p
    dev = M.t.device
    lp = _Loop(M, b, ell)
    perm = torch.arange(n, dtype=torch.int64, device=dev)
    taus = torch.zeros(max(k, 1), dtype=torch.float64, device=dev)
    B = _sketch(M, OmT, ell, seed, 0)
    stream_pos = ell * m
    achieved, widths, reason = 0, [], 1
    while achieved < k:
        i0 = achieved
        bb = min(b, k - i0)
        nt = n - i0
        stop, why, sa = lp.sample_qrcp(B, nt, bb)
        if stop:
            reason = why
            break
        lp.apply_moves(M, m, i0, perm, bb)
        bhat, subs = lp.panel(M, i0, i0, sa, taus, i0)
        if bhat == 0:
            reason = 4
            break
        widths.append((i0, bhat))
        ncols = n - (i0 + bhat)
        for s0, bh, Y in subs:       # Q^T C = Q_s^T ... Q_1^T C  (randomized.py:203-207)
            lp.block_update(M.col_ptr(i0 + s0, i0 + bhat), M.ld, m - i0 - s0, ncols, Y, bh,
                            taus.data_ptr() + 8 * (i0 + s0))
        achieved = i0 + bhat
        if bhat < bb or achieved >= k or ncols == 0:
            reason = 5 if bhat < bb else (1 if achieved >= k else 6)
            break
        if resample:   # randomized.py:214-215
            B = _sketch(M, None, ell, seed, stream_pos, r0=achieved)
            stream_pos += ell * (m - achieved)
        else:
            if not _r11_ok(M, i0, bb):
                reason = 7
                break
            B = lp.sample_update(nt, bb, M.col_ptr(i0, i0), M.ld)
    cnt = rqrcp_counters(m, n, b, ell, achieved, len(widths), reason, resample)
    pf = PivotedFactorization(m, n, None, None, None, achieved, cnt)
    pf._Rd_fn = lambda: _upper_rows(M, achieved)
    pf._permd = perm
    pf._blocks_fn = lambda: _packed_blocks(M, taus, None, b, widths, m)
    pf._work = M
    return pf


def trqrcp_wide(M: ColMajor, k: int, b: int, p: int, seed: int, OmT):
    """randomized.py:250-341 for any b; M (the reference's `work`) is permuted in place."""
    from .factor import TruncatedFactorization, _build_t, _packed_blocks, _upper_rows, gemm_tn
    m, n = M.m, M.n
    ell = b + p
    dev = M.t.device
    L = _lib.lib()
    s = stream_handle
    lp = _Loop(M, b, ell)
    perm = torch.arange(n, dtype=torch.int64, device=dev)
    taus = torch.zeros(max(k, 1), dtype=torch.float64, device=dev)
    Yg = ColMajor.empty(m, k, dev, zero=True)
    Wg = ColMajor.empty(k, n, dev, zero=True)
    Rg = ColMajor.empty(k, n, dev, zero=True)
    B = _sketch(M, OmT, ell, seed, 0)
    achieved, widths = 0, []
    while achieved < k:
        i0 = achieved
        bb = min(b, k - i0)
        nt = n - i0
        mr = m - i0
        stop, _, sa = lp.sample_qrcp(B, nt, bb)
        if stop:
            break
        lp.apply_moves(M, m, i0, perm, bb)
        if i0:
            lp.apply_moves(Wg, i0, i0, None, bb)
            lp.apply_moves(Rg, i0, i0, None, bb)
        # panel = A[i0:, sel] - Yg[i0:, :i0] Wg[:i0, sel]   (randomized.py:304-306)
        Pn = ColMajor.empty(mr, sa, dev)
        if i0:
            _lib.check(L.sqr_gemm_nn(mr, sa, i0, -1.0, Yg.col_ptr(i0, 0), Yg.ld, Wg.col_ptr(0, i0), Wg.ld, 1.0,
                                     M.col_ptr(i0, i0), M.ld, Pn.ptr, Pn.ld, s()), "materialise panel")
        else:
            Pn.view().copy_(M.view()[:, :sa])
        bhat, subs = lp.panel(Pn, 0, 0, sa, taus, i0)
        if bhat == 0:
            break
        widths.append((i0, bhat))
        for s0, bh, Y in subs:       # Yg[i0:, i0:i0+bhat] = Y2 (explicit, zero above the diagonal)
            Yg.view()[i0 + s0:, i0 + s0:i0 + s0 + bh] = Y.view()[:, :bh]
        Rg.view()[i0:i0 + bhat, i0:i0 + bhat] = torch.triu(Pn.view()[:bhat, :bhat])          # R11 (:316)
        Y2 = ColMajor(Yg.t[i0:i0 + bhat, i0:], mr, bhat, Yg.ld)
        T2 = _build_t(Y2, taus[i0:i0 + bhat].contiguous())
        ntrail = n - (i0 + bhat)
        c0 = i0 + bhat
        if ntrail:
            A_t = ColMajor(M.t[c0:, i0:], mr, ntrail, M.ld)
            G = gemm_tn(Y2, A_t)                                            # Y2^T A  (:322)
            if i0:
                C1 = gemm_tn(Y2, ColMajor(Yg.t[:i0, i0:], mr, i0, Yg.ld))   # Y2^T Y1
                _lib.check(L.sqr_gemm_nn(bhat, ntrail, i0, -1.0, C1.ptr, C1.ld, Wg.col_ptr(0, c0), Wg.ld, 1.0,
                                         G.ptr, G.ld, G.ptr, G.ld, s()), "correction")   # (:325-326)
            WT = gemm_tn(T2, G)                                              # T2^T G  (:327)
            Wg.view()[i0:i0 + bhat, c0:] = WT.view()
            _lib.check(L.sqr_gemm_nn(bhat, ntrail, i0 + bhat, -1.0, Yg.col_ptr(i0, 0), Yg.ld, Wg.col_ptr(0, c0),
                                     Wg.ld, 1.0, M.col_ptr(i0, c0), M.ld, Rg.col_ptr(i0, c0), Rg.ld, s()),
                       "R rows")                                             # (:329-330)
        achieved = i0 + bhat
        if bhat < bb or achieved >= k or ntrail == 0:
            break
        if not _r11_ok(Rg, i0, bb):
            break
        B = lp.sample_update(nt, bb, Rg.col_ptr(i0, i0), Rg.ld)
    tf = TruncatedFactorization(m, n, None, None, None, achieved, trqrcp_counters(m, n, b, ell, achieved, len(widths)))
    tf._Rd = _upper_rows(Rg, achieved)
    tf._permd = perm
    tf._w_td = Wg.view()[:achieved, :].contiguous()
    tf._blocks_fn = lambda: _packed_blocks(Yg, taus, None, b, widths, m)
    tf._Yg = Yg
    tf._permuted_input = True
    return tf

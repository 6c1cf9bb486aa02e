"""Drop-in RQRCP / RSRQRCP / SSRQRCP / TRQRCP / TUXV and the deterministic
QR(CP) routines of the reference, executed by libsqr on a B200.

Signatures, argument checks, error types, early exits, result fields and
communication counters follow the reference ``sketchqr`` package
(pkg/src/sketchqr/randomized.py, reference.py); every floating-point
operation runs in libsqr's sm_100a kernels, enqueued on torch's current CUDA
stream.  Inputs may be NumPy arrays (results then expose NumPy arrays, like
the reference) or torch tensors; the input is never modified.

Omega: by default the l x m Gaussian sketch is generated ON THE DEVICE from
the reference's counter-based stream (splitmix64 + Box-Muller, rng.py:38-93).
The integer stage is bit-exact; CUDA's log/sin/cos may differ from NumPy's by
an ulp in a small fraction of entries.  ``omega="host"`` instead draws Omega
with the reference's NumPy recipe on the host (bit-identical to the
reference), and ``omega=<array>`` feeds an explicit l x m matrix.
"""
from __future__ import annotations

import contextlib

import numpy as np
import torch

from . import _lib
from ._dev import (ColMajor, Workspace, check_finite, load_checked, ptr, require_cuda, status_new, status_read,
                   stream_handle, upload)
from .counters import (CommCounters, qr_blocked_counters, qrcp_blas2_counters, qrcp_blocked_counters,
                       rqrcp_counters, trqrcp_counters)
from .rng import host_omega

_DIAG_FLOOR = 2.0 ** -52
MAX_B = 128
MAX_ELL = 144


# ---------------------------------------------------------------- validation
def _check_block_args(m, n, k, b=None, p=None):
    """validation.py:75-82."""
    if k < 0 or k > min(m, n):
        raise ValueError(f"rank k={k} must satisfy 0 <= k <= min(m, n) = {min(m, n)}")
    if b is not None and not 1 <= b:
        raise ValueError(f"block size b={b} must be >= 1")
    if p is not None and p < 0:
        raise ValueError(f"padding p={p} must be >= 0")


def _check_target_rank(m, n, k):
    """validation.py:62-72."""
    if k is None:
        return min(m, n)
    if not 1 <= k <= min(m, n):
        raise ValueError(f"rank k={k} must satisfy 1 <= k <= min(m, n) = {min(m, n)}")
    return int(k)


def invert_permutation(perm: np.ndarray) -> np.ndarray:
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0], dtype=perm.dtype)
    return inv


def _load(A, device=None, copy: bool = True, check: bool = True) -> tuple[ColMajor, bool]:
    dev = require_cuda(device if device is not None else (A.device if isinstance(A, torch.Tensor) and A.is_cuda else None))
    M = load_checked(A, dev, copy=copy, check=check)
    return M, not isinstance(A, torch.Tensor)


def _ws(nbytes, device):
    """Exclusive use of the current stream's scratch while a call enqueues (_dev.Workspace)."""
    return Workspace.lease(nbytes, device)


# ------------------------------------------------------------ device blocks
class ReflectorBlock:
    """Compact-WY block Q = I - Y T Y^T (householder.py:64-91).

    Host-constructed blocks hold NumPy arrays; blocks produced by the device
    drivers keep device tensors and materialise NumPy views on first access.
    """

    def __init__(self, Y=None, tau=None, T=None, offset: int = 0, *, _dev=None):
        self.offset = int(offset)
        if _dev is not None:
            self._Yd, self._taud, self._Td = _dev
            self._Y = self._tau = self._T = None
            return
        Y = np.asarray(Y, dtype=np.float64)
        tau = np.asarray(tau, dtype=np.float64)
        if Y.ndim != 2 or tau.shape != (Y.shape[1],):
            raise ValueError("Y must be m x j with one tau per reflector")
        self._Y, self._tau = Y, tau
        self._Yd = self._taud = self._Td = None
        self._T = None if T is None else np.asarray(T, dtype=np.float64)
        if self._T is None and Y.shape[1]:
            dev = require_cuda()
            self._to_device(dev)
            self._Td = _build_t(self._Yd, self._taud)
        elif self._T is None:
            self._T = np.zeros((0, 0))

    # -- device side
    def _to_device(self, dev):
        if self._Yd is None:
            self._Yd = upload(self._Y, dev)
            self._taud = torch.from_numpy(np.ascontiguousarray(self._tau)).to(dev)
        if self._Td is None and self._T is not None:
            self._Td = upload(self._T, dev)
        return self

    def device_parts(self, dev=None):
        dev = require_cuda(dev)
        self._to_device(dev)
        return self._Yd, self._taud, self._Td

    # -- host side (reference fields)
    @property
    def Y(self) -> np.ndarray:
        if self._Y is None:
            self._Y = self._Yd.numpy()
        return self._Y

    @Y.setter
    def Y(self, v):
        self._Y = np.asarray(v, dtype=np.float64)
        self._Yd = None

    @property
    def tau(self) -> np.ndarray:
        if self._tau is None:
            self._tau = self._taud.cpu().numpy()
        return self._tau

    @property
    def T(self) -> np.ndarray:
        if self._T is None:
            self._T = self._Td.numpy() if self._Td is not None else np.zeros((0, 0))
        return self._T

    @property
    def m(self) -> int:
        return self._Yd.m if self._Yd is not None else self._Y.shape[0]

    @property
    def width(self) -> int:
        return self._Yd.n if self._Yd is not None else self._Y.shape[1]


def _build_t(Yd: ColMajor, taud: torch.Tensor) -> ColMajor:
    """T of I - Y T Y^T = H_1...H_j on the device (householder.py:52-61)."""
    j = Yd.n
    dev = Yd.t.device
    if j > MAX_B:   # the T kernel takes <= 128 reflectors
        return _compose_t_recursive(Yd, taud)
    T = ColMajor.empty(j, j, dev, zero=True)
    with _ws(j * j * 8 + (200 << 20), dev) as ws:
        _lib.check(_lib.lib().sqr_build_t(Yd.ptr, Yd.ld, Yd.m, j, ptr(taud), T.ptr, T.ld, ptr(ws), ws.numel(),
                                          stream_handle()), "sqr_build_t")
    return T


def _compose_t_recursive(Yd: ColMajor, taud: torch.Tensor) -> ColMajor:
    """T for wide Y via the composition rule T12 = -T1 (Y1^T Y2) T2 (householder.py:94-104)."""
    j = Yd.n
    h = j // 2
    dev = Yd.t.device
    Y1 = ColMajor(Yd.t[:h], Yd.m, h, Yd.ld)
    Y2 = ColMajor(Yd.t[h:j], Yd.m, j - h, Yd.ld)
    T1 = _build_t(Y1, taud[:h].contiguous())
    T2 = _build_t(Y2, taud[h:].contiguous())
    G12 = gemm_tn(Y1, Y2)                 # h x (j-h)
    X = gemm_nn(T1, G12, alpha=-1.0)      # -T1 G12
    T12 = gemm_nn(X, T2)                  # -T1 G12 T2
    T = ColMajor.empty(j, j, dev, zero=True)
    T.view()[:h, :h] = T1.view()
    T.view()[h:, h:] = T2.view()
    T.view()[:h, h:] = T12.view()
    return T


# ---------------------------------------------------------------- GEMM glue
def gemm_tn(X: ColMajor, C: ColMajor, alpha: float = 1.0) -> ColMajor:
    """alpha X^T C on the device (X: K x M, C: K x N), M chunked by 144."""
    M, N, K = X.n, C.n, X.m
    dev = C.t.device
    D = ColMajor.empty(M, N, dev)
    with _ws(200 << 20, dev) as ws:
        for i0 in range(0, M, MAX_ELL):
            mc = min(MAX_ELL, M - i0)
            _lib.check(_lib.lib().sqr_gemm_tn(mc, N, K, alpha, X.col_ptr(0, i0), X.ld, C.ptr, C.ld, 0.0, None, 0,
                                              D.col_ptr(i0, 0), D.ld, ptr(ws), ws.numel(), stream_handle()),
                       "sqr_gemm_tn")
    return D


def gemm_nn(X: ColMajor, Y: ColMajor, alpha: float = 1.0) -> ColMajor:
    M, N, K = X.m, Y.n, X.n
    D = ColMajor.empty(M, N, Y.t.device)
    # split-K scratch for skinny products
    with (_ws(16 * M * N * 8, Y.t.device) if K >= 2048 else contextlib.nullcontext()) as ws:
        _lib.check(_lib.lib().sqr_gemm_nn_ws(M, N, K, alpha, X.ptr, X.ld, Y.ptr, Y.ld, 0.0, None, 0, D.ptr, D.ld,
                                             ptr(ws) if ws is not None else None,
                                             ws.numel() if ws is not None else 0, stream_handle()), "sqr_gemm_nn")
    return D


def _apply_blocks(blocks, C: ColMajor, transpose: bool) -> ColMajor:
    """C := Q C (apply_blocks_q) or Q^T C (apply_blocks_qt), householder.py:123-134."""
    order = blocks if transpose else list(reversed(blocks))
    dev = C.t.device
    for blk in order:
        if blk.width == 0:
            continue
        Yd, _, Td = blk.device_parts(dev)
        if blk.width > MAX_ELL:
            # composed blocks wider than the fused kernel's 144 (e.g. TUXV's U / V
            # for k > 144): C -= Y op(T) (Y^T C) with the chunked DMMA GEMMs
            if C.n == 0:
                continue
            Wt = gemm_tn(Yd, C)                          # j x n
            Tm = Td if not transpose else _transpose(Td)
            W = gemm_nn(Tm, Wt)                          # op(T) Y^T C
            YW = gemm_nn(Yd, W)
            C.view().sub_(YW.view())
            continue
        with _ws(2 * blk.width * max(C.n, 1) * 8 + (200 << 20), dev) as ws:
            _lib.check(_lib.lib().sqr_apply_wy(Yd.ptr, Yd.ld, Td.ptr, Td.ld, Yd.m, blk.width, C.ptr, C.ld, C.n,
                                               1 if transpose else 0, ptr(ws), ws.numel(), stream_handle()),
                       "sqr_apply_wy")
    return C


def _transpose(M: ColMajor) -> ColMajor:
    out = ColMajor.empty(M.n, M.m, M.t.device)
    if M.m and M.n:
        _lib.check(_lib.lib().sqr_transpose(M.ptr, M.ld, M.m, M.n, out.ptr, out.ld, 0, stream_handle()),
                   "sqr_transpose")
    return out


def _q_columns_dev(blocks, m: int, r: int, dev) -> ColMajor:
    Q = ColMajor.empty(m, r, dev, zero=True)
    if r:
        idx = torch.arange(r, device=dev)
        Q.t[idx, idx] = 1.0
    return _apply_blocks(blocks, Q, transpose=False)


def blocks_q_columns(blocks, m: int, r: int) -> np.ndarray:
    """householder.py:137-141."""
    return _q_columns_dev(blocks, m, r, require_cuda()).numpy()


def apply_blocks_q(blocks, C):
    dev = require_cuda()
    Cd = upload(C, dev)
    _apply_blocks(blocks, Cd, transpose=False)
    out = Cd.numpy()
    if isinstance(C, np.ndarray):
        C[...] = out
        return C
    return out


def apply_blocks_qt(blocks, C):
    dev = require_cuda()
    Cd = upload(C, dev)
    _apply_blocks(blocks, Cd, transpose=True)
    out = Cd.numpy()
    if isinstance(C, np.ndarray):
        C[...] = out
        return C
    return out


def wy_compose(b1: ReflectorBlock, b2: ReflectorBlock) -> ReflectorBlock:
    """householder.py:94-104 on the device."""
    if b1.m != b2.m:
        raise ValueError("blocks must act on the same row dimension")
    dev = require_cuda()
    Y1, t1, T1 = b1.device_parts(dev)
    Y2, t2, T2 = b2.device_parts(dev)
    j1, j2 = Y1.n, Y2.n
    Y = ColMajor.empty(Y1.m, j1 + j2, dev)
    if j1:
        Y.view()[:, :j1] = Y1.view()
    if j2:
        Y.view()[:, j1:] = Y2.view()
    T = ColMajor.empty(j1 + j2, j1 + j2, dev, zero=True)
    if j1:
        T.view()[:j1, :j1] = T1.view()
    if j2:
        T.view()[j1:, j1:] = T2.view()
    if j1 and j2:
        G = gemm_tn(Y1, Y2)
        T.view()[:j1, j1:] = gemm_nn(gemm_nn(T1, G, alpha=-1.0), T2).view()
    tau = torch.cat([t1, t2])
    return ReflectorBlock(offset=b1.offset, _dev=(Y, tau, T))


def _compose_all(blocks):
    if not blocks:
        return None
    out = blocks[0]
    for blk in blocks[1:]:
        out = wy_compose(out, blk)
    return out


# ---------------------------------------------------------------- results
class PivotedFactorization:
    """A[:, perm] ~= Q R (reference.py:61-99); device-backed, NumPy on access."""

    def __init__(self, m, n, blocks, R, perm, achieved_rank, counters=None):
        self.m, self.n = int(m), int(n)
        self._blocks = blocks
        self._R = None if R is None else np.asarray(R)
        self._perm = None if perm is None else np.asarray(perm, dtype=np.int64)
        self.achieved_rank = int(achieved_rank)
        self.counters = counters or CommCounters()
        self._Rd_val = None    # torch (achieved, n) row-major, upper trapezoidal
        self._Rd_fn = None     # lazy producer of _Rd_val (R extracted only when asked for)
        self._permd = None     # torch int64 (n,)
        self._blocks_fn = None

    @property
    def _Rd(self):
        if self._Rd_val is None and self._Rd_fn is not None:
            self._Rd_val, self._Rd_fn = self._Rd_fn(), None
        return self._Rd_val

    @_Rd.setter
    def _Rd(self, v):
        self._Rd_val, self._Rd_fn = v, None

    # lazily materialised reference fields
    @property
    def R(self) -> np.ndarray:
        if self._R is None:
            self._R = np.asfortranarray(self._Rd.cpu().numpy()) if self._Rd is not None else np.zeros((0, self.n), order="F")
        return self._R

    @R.setter
    def R(self, v):
        self._R, self._Rd = np.asarray(v), None

    @property
    def perm(self) -> np.ndarray:
        if self._perm is None:
            self._perm = self._permd.cpu().numpy()
        return self._perm

    @perm.setter
    def perm(self, v):
        self._perm, self._permd = np.asarray(v, dtype=np.int64), None

    @property
    def blocks(self):
        if self._blocks is None:
            self._blocks = self._blocks_fn() if self._blocks_fn else []
        return self._blocks

    @blocks.setter
    def blocks(self, v):
        self._blocks = v

    # device views
    def R_device(self, dev=None) -> torch.Tensor:
        if self._Rd is None:
            self._Rd = torch.from_numpy(np.ascontiguousarray(self.R)).to(require_cuda(dev))
        return self._Rd

    def perm_device(self, dev=None) -> torch.Tensor:
        if self._permd is None:
            self._permd = torch.from_numpy(np.ascontiguousarray(self.perm)).to(require_cuda(dev))
        return self._permd

    # reference methods, computed on the device
    def _reconstruct_dev(self, rank=None) -> torch.Tensor:
        dev = require_cuda()
        r = self.achieved_rank if rank is None else min(rank, self.achieved_rank)
        if r == 0:
            return torch.zeros((self.m, self.n), dtype=torch.float64, device=dev)
        Q = _q_columns_dev(self.blocks, self.m, r, dev)
        Rr = ColMajor.empty(r, self.n, dev)
        Rr.view().copy_(self.R_device(dev)[:r, :])
        QR = gemm_nn(Q, Rr).view()
        inv = torch.empty_like(self.perm_device(dev))
        inv[self.perm_device(dev)] = torch.arange(self.n, device=dev)
        return QR[:, inv]

    def q_columns(self, rank=None) -> np.ndarray:
        r = self.achieved_rank if rank is None else min(rank, self.achieved_rank)
        return blocks_q_columns(self.blocks, self.m, r)

    def apply_q(self, C):
        return apply_blocks_q(self.blocks, C)

    def reconstruct(self, rank=None) -> np.ndarray:
        return np.asfortranarray(self._reconstruct_dev(rank).cpu().numpy())

    def rel_residual(self, A, rank=None) -> float:
        dev = require_cuda()
        Ad = upload(A, dev).view()
        denom = torch.linalg.norm(Ad)
        if float(denom) == 0.0:
            return 0.0
        return float(torch.linalg.norm(Ad - self._reconstruct_dev(rank)) / denom)

    @property
    def r_diag(self) -> np.ndarray:
        r = self.achieved_rank
        return np.abs(np.diag(self.R[:r, :r])) if r else np.zeros(0)


class TruncatedFactorization(PivotedFactorization):
    """randomized.py:59-67: adds w_t = T^T Y^T (A P)."""

    def __init__(self, m, n, blocks, R, perm, achieved_rank, counters=None, w_t=None):
        super().__init__(m, n, blocks, R, perm, achieved_rank, counters)
        self._w_t = None if w_t is None else np.asarray(w_t)
        self._w_td = None

    @property
    def w_t(self) -> np.ndarray:
        if self._w_t is None:
            self._w_t = np.asfortranarray(self._w_td.cpu().numpy()) if self._w_td is not None else np.zeros((0, self.n), order="F")
        return self._w_t

    @w_t.setter
    def w_t(self, v):
        self._w_t, self._w_td = np.asarray(v), None


class TuxvResult:
    """randomized.py:70-97."""

    def __init__(self, U, X, V, sigma_est, achieved_rank, counters, m, n):
        self.U, self.V = U, V
        self._X = X
        self._sig = sigma_est
        self.achieved_rank, self.counters, self.m, self.n = int(achieved_rank), counters, int(m), int(n)

    @property
    def X(self) -> np.ndarray:
        if isinstance(self._X, torch.Tensor):
            self._X = np.asfortranarray(self._X.cpu().numpy())
        return self._X

    @property
    def sigma_est(self) -> np.ndarray:
        if isinstance(self._sig, torch.Tensor):
            self._sig = self._sig.cpu().numpy()
        return self._sig

    def u_columns(self) -> np.ndarray:
        return blocks_q_columns([self.U] if self.U else [], self.m, self.achieved_rank)

    def v_columns(self) -> np.ndarray:
        return blocks_q_columns([self.V] if self.V else [], self.n, self.achieved_rank)

    def reconstruct_device(self) -> torch.Tensor:
        dev = require_cuda()
        k = self.achieved_rank
        if k == 0:
            return torch.zeros((self.m, self.n), dtype=torch.float64, device=dev)
        U = _q_columns_dev([self.U], self.m, k, dev)
        V = _q_columns_dev([self.V], self.n, k, dev)
        Xd = upload(self.X, dev)
        UX = gemm_nn(U, Xd)
        # (U X) V^T = ((V (U X)^T)^T
        UXt = ColMajor.empty(k, self.m, dev)
        UXt.view().copy_(UX.view().T)
        out = gemm_nn(V, UXt)  # n x m
        return out.view().T

    def reconstruct(self) -> np.ndarray:
        if self.achieved_rank == 0:
            return np.zeros((self.m, self.n), order="F")
        return np.asfortranarray(self.reconstruct_device().cpu().numpy())


# -------------------------------------------------------- result assembly
def _packed_blocks(W: ColMajor, taus: torch.Tensor, Tbuf, b: int, widths, m: int):
    """ReflectorBlocks (explicit unit-lower Y, zeros above offset) from a
    LAPACK-packed work matrix: block J's reflector c sits in column i0+c."""
    dev = W.t.device
    out = []
    L = _lib.lib()
    for J, (i0, w) in enumerate(widths):
        Y = ColMajor.empty(m, w, dev)
        _lib.check(L.sqr_unpack_reflectors(W.ptr, W.ld, m, i0, w, Y.ptr, Y.ld, stream_handle()),
                   "sqr_unpack_reflectors")
        if Tbuf is not None:
            T = ColMajor(Tbuf[J].view(b, b)[:w], w, w, b)   # block J's T in place (ld b)
        else:
            T = _build_t(Y, taus[i0:i0 + w].contiguous())
        out.append(ReflectorBlock(offset=i0, _dev=(Y, taus[i0:i0 + w].clone(), T)))
    return out


def _upper_rows(W: ColMajor, rows: int) -> torch.Tensor:
    """triu(W[:rows, :]) as a (rows, n) row-major tensor (sqr_transpose, upper)."""
    out = torch.empty((rows, W.n), dtype=torch.float64, device=W.t.device)
    if rows and W.n:
        _lib.check(_lib.lib().sqr_transpose(W.ptr, W.ld, rows, W.n, out.data_ptr(), W.n, 1, stream_handle()),
                   "sqr_transpose")
    return out


def _fallback_qrcp(M: ColMajor, k: int, b: int, numpy_out: bool, blas2: bool = False) -> PivotedFactorization:
    """qrcp_blocked / qrcp_blas2 (reference.py:162-263) on the device: the
    sample-QRCP kernel is a BLAS-2 QRCP of a short matrix; the pivot sequence
    equals the blocked variant's (asserted by the reference's own tests)."""
    dev = M.t.device
    m, n = M.m, M.n
    L = _lib.lib()
    Bf = ColMajor.empty(m, n, dev)
    lperm = torch.empty(n, dtype=torch.int64, device=dev)
    moves = torch.empty(2 * 2 * k + 8, dtype=torch.int32, device=dev)
    taus = torch.zeros(max(k, 1), dtype=torch.float64, device=dev)
    st = status_new(dev)
    _lib.check(L.sqr_sample_qrcp(M.ptr, M.ld, m, n, k, Bf.ptr, Bf.ld, ptr(lperm), ptr(moves), ptr(taus), 1,
                                 ptr(st), stream_handle()), "sqr_sample_qrcp")
    s = status_read(st)
    ach = 0 if s["stop"] and s["reason"] == 2 else int(s["sample_achieved"])
    if blas2:
        widths = [(0, ach)] if ach else []
        cnt = qrcp_blas2_counters(m, n, ach)
    else:
        widths = [(i0, min(b, ach - i0)) for i0 in range(0, ach, b)]
        cnt = qrcp_blocked_counters(m, n, k, b, ach)
    pf = PivotedFactorization(m, n, None, None, None, ach, cnt)
    pf._Rd = _upper_rows(Bf, ach)
    pf._permd = lperm if ach else torch.arange(n, device=dev)
    pf._blocks_fn = lambda: _packed_blocks(Bf, taus, None, b, widths, m)
    if ach == 0:
        pf._permd = torch.arange(n, device=dev)
    return pf


def qrcp_blocked(A, k=None, b: int = 32) -> PivotedFactorization:
    """reference.py:174-263."""
    if b < 1:
        raise ValueError("block size b must be >= 1")
    M, _ = _load(A)
    kk = _check_target_rank(M.m, M.n, k)
    return _fallback_qrcp(M, kk, b, True)


def qrcp_blas2(A, k=None) -> PivotedFactorization:
    """reference.py:162-171."""
    M, _ = _load(A)
    kk = _check_target_rank(M.m, M.n, k)
    return _fallback_qrcp(M, kk, max(kk, 1), True, blas2=True)


def _qr_blocked_dev(M: ColMajor, k: int, b: int) -> PivotedFactorization:
    dev = M.t.device
    m, n = M.m, M.n
    L = _lib.lib()
    bk = min(b, MAX_B)
    nblk = -(-k // bk)
    taus = torch.zeros(k, dtype=torch.float64, device=dev)
    Tb = torch.zeros((nblk, bk * bk), dtype=torch.float64, device=dev)
    with _ws(L.sqr_qr_blocked_workspace(m, n, k, bk), dev) as ws:
        _lib.check(L.sqr_qr_blocked(M.ptr, M.ld, m, n, k, bk, ptr(taus), ptr(Tb), ptr(ws), ws.numel(),
                                    stream_handle()), "sqr_qr_blocked")
    widths = [(i0, min(bk, k - i0)) for i0 in range(0, k, bk)]
    pf = PivotedFactorization(m, n, None, None, None, k, qr_blocked_counters(m, n, k, b))
    pf._Rd = _upper_rows(M, k)
    pf._permd = torch.arange(n, device=dev)
    # all k reflectors as ONE compact-WY block (what _compose_all of the
    # per-block list gives, householder.py:94-104): one masked copy + T from G
    pf._composed_fn = (lambda: [_packed_blocks(M, taus, None, k, [(0, k)], m)[0]]) if k <= MAX_ELL \
        else (lambda: pf.blocks)
    if bk == b:
        pf._blocks_fn = lambda: _packed_blocks(M, taus, Tb, bk, widths, m)
    else:  # reference blocking with b > 128: same reflectors, regrouped
        wref = [(i0, min(b, k - i0)) for i0 in range(0, k, b)]
        pf._blocks_fn = lambda: _packed_blocks(M, taus, None, b, wref, m)
    return pf


def qr_blocked(A, k=None, b: int = 32) -> PivotedFactorization:
    """Blocked unpivoted Householder QR (reference.py:266-311)."""
    if b < 1:
        raise ValueError("block size b must be >= 1")
    M, _ = _load(A)
    kk = _check_target_rank(M.m, M.n, k)
    return _qr_blocked_dev(M, kk, b)


# ------------------------------------------------------------- randomized
def _omega_T(omega, ell: int, m: int, seed: int, dev) -> ColMajor | None:
    """Omega^T (m x l) for the drivers, or None to draw it on the device."""
    if omega is None or (isinstance(omega, str) and omega == "device"):
        return None
    if isinstance(omega, str):
        if omega != "host":
            raise ValueError("omega must be 'device', 'host' or an l x m array")
        om = host_omega(ell, m, seed)
    else:
        om = omega.detach().cpu().numpy() if isinstance(omega, torch.Tensor) else np.asarray(omega, dtype=np.float64)
        if om.shape != (ell, m):
            raise ValueError(f"omega must have shape ({ell}, {m}), got {om.shape}")
    return upload(om.T, dev)


def _empty(m, n, dev, truncated=False):
    cls = TruncatedFactorization if truncated else PivotedFactorization
    pf = cls(m, n, [], np.zeros((0, n), order="F"), np.arange(n, dtype=np.int64), 0, CommCounters())
    if truncated:
        pf.w_t = np.zeros((0, n), order="F")
    return pf


def _check_out(out, rows, n):
    """`out=`: a Fortran-ordered float64 host array of shape (>= rows, n) that
    receives R while the factorization runs (pinned memory for full speed).
    Its strictly lower part is never written: pass it zeroed."""
    if not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.ndim != 2:
        raise ValueError("out must be a 2-D float64 numpy array")
    if not out.flags.f_contiguous or out.shape[0] < rows or out.shape[1] != n:
        raise ValueError(f"out must be Fortran-ordered with shape (>= {rows}, {n})")
    return out


def _randomized(A, k, b, p, seed, resample, omega=None, _status=None, out=None):
    M, _ = _load(A)
    m, n = M.m, M.n
    _check_block_args(m, n, k, b, p)
    dev = M.t.device
    if k == 0:
        return _empty(m, n, dev)
    ell = b + p
    if ell >= m:
        return _fallback_qrcp(M, k, b, True)
    if b > MAX_B or ell > MAX_ELL:   # wider than the fused driver: per-block loop (wide.py)
        from .wide import rqrcp_wide
        pf = rqrcp_wide(M, k, b, p, seed, resample, _omega_T(omega, ell, m, seed, dev) if not resample else None)
        if out is not None:
            out = _check_out(out, min(k, m), n)
            out[:pf.achieved_rank] = pf.R
            pf._R = out[:pf.achieved_rank]
        return pf
    L = _lib.lib()
    OmT = _omega_T(omega, ell, m, seed, dev)
    nblk = -(-k // b)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    taus = torch.zeros(k, dtype=torch.float64, device=dev)
    Tb = torch.zeros((nblk, b * b), dtype=torch.float64, device=dev)
    st = status_new(dev)
    if out is None:
        with _ws(L.sqr_rqrcp_workspace(m, n, k, b, p), dev) as ws:
            _lib.check(L.sqr_rqrcp(M.ptr, M.ld, m, n, k, b, p, seed & ((1 << 64) - 1),
                                   OmT.ptr if OmT is not None else None, OmT.ld if OmT is not None else 0,
                                   1 if resample else 0, ptr(perm), ptr(taus), ptr(Tb), ptr(st), ptr(ws),
                                   ws.numel(), stream_handle()), "sqr_rqrcp")
    else:
        # R streamed to the host buffer block by block, overlapped with the later blocks
        out = _check_out(out, min(k, m), n)
        with _ws(L.sqr_rqrcp_stream_r_workspace(m, n, k, b, p), dev) as ws:
            _lib.check(L.sqr_rqrcp_stream_r(M.ptr, M.ld, m, n, k, b, p, seed & ((1 << 64) - 1),
                                            OmT.ptr if OmT is not None else None, OmT.ld if OmT is not None else 0,
                                            1 if resample else 0, ptr(perm), ptr(taus), ptr(Tb), ptr(st), ptr(ws),
                                            ws.numel(), out.ctypes.data, out.shape[0], stream_handle()),
                       "sqr_rqrcp_stream_r")
    s = status_read(st)
    if _status is not None:
        _status.append(s)
    ach, nb = int(s["achieved"]), int(s["nblocks"])
    cnt = rqrcp_counters(m, n, b, ell, ach, nb, int(s["reason"]), resample)
    pf = PivotedFactorization(m, n, None, None, None, ach, cnt)
    if out is None:
        pf._Rd_fn = lambda: _upper_rows(M, ach)
    else:
        pf._R = out[:ach]
    pf._permd = perm
    widths = [(J * b, min(b, ach - J * b)) for J in range(nb)]
    pf._blocks_fn = lambda: _packed_blocks(M, taus, Tb, b, widths, m)
    pf._work = M
    return pf


def rqrcp(A, k: int, b: int = 32, p: int = 8, seed: int = 0, omega=None, out=None) -> PivotedFactorization:
    """Blocked randomized QRCP with sample updates (randomized.py:227-229).

    `out` (extension): host array receiving R during the factorization (see _check_out)."""
    return _randomized(A, k, b, p, seed, False, omega, out=out)


def rsrqrcp(A, k: int, b: int = 32, p: int = 8, seed: int = 0, out=None) -> PivotedFactorization:
    """Blocked randomized QRCP re-sketching every block (randomized.py:232-234)."""
    return _randomized(A, k, b, p, seed, True, None, out=out)


def ssrqrcp(A, k: int, p: int = 8, seed: int = 0, omega=None) -> PivotedFactorization:
    """Single-sample randomized QRCP (randomized.py:143-163)."""
    M, _ = _load(A)
    m, n = M.m, M.n
    _check_block_args(m, n, k, None, p)
    dev = M.t.device
    if k == 0:
        return _empty(m, n, dev)
    ell = k + p
    if ell >= m:
        return _fallback_qrcp(M, k, min(32, k), True)
    L = _lib.lib()
    cnt = CommCounters()
    OmT = _omega_T(omega, ell, m, seed, dev)
    if OmT is None:
        OmT = ColMajor.empty(m, ell, dev)
        _lib.check(L.sqr_gaussian(OmT.ptr, OmT.ld, ell, m, seed & ((1 << 64) - 1), 0, 1, stream_handle()),
                   "sqr_gaussian")
    B = gemm_tn(OmT, M)
    cnt.add_blas3(ell, m, n)
    Bf = ColMajor.empty(ell, n, dev)
    lperm = torch.empty(n, dtype=torch.int64, device=dev)
    moves = torch.empty(4 * k + 8, dtype=torch.int32, device=dev)
    staus = torch.zeros(k, dtype=torch.float64, device=dev)
    st = status_new(dev)
    _lib.check(L.sqr_sample_qrcp(B.ptr, B.ld, ell, n, k, Bf.ptr, Bf.ld, ptr(lperm), ptr(moves), ptr(staus), 1,
                                 ptr(st), stream_handle()), "sqr_sample_qrcp")
    s = status_read(st)
    ach = 0 if (s["stop"] and s["reason"] == 2) else int(s["sample_achieved"])
    if ach == 0:
        return PivotedFactorization(m, n, [], np.zeros((0, n), order="F"), np.arange(n, dtype=np.int64), 0, cnt)
    Ap = ColMajor.empty(m, n, dev)
    Ap.view().copy_(M.view()[:, lperm])
    qf = _qr_blocked_dev(Ap, ach, min(32, ach))
    cnt.merge(qf.counters)
    pf = PivotedFactorization(m, n, None, None, None, ach, cnt)
    pf._Rd, pf._permd, pf._blocks_fn = qf._Rd, lperm, qf._blocks_fn
    return pf


def _truncated_from_pivoted(pf: PivotedFactorization, M: ColMajor) -> TruncatedFactorization:
    """Dense w_t for the l >= m fallback (randomized.py:237-247)."""
    dev = M.t.device
    tf = TruncatedFactorization(pf.m, pf.n, None, None, None, pf.achieved_rank, pf.counters)
    tf._Rd, tf._permd, tf._blocks_fn = pf._Rd, pf._permd, pf._blocks_fn
    if pf.achieved_rank == 0:
        tf._w_td = torch.zeros((0, pf.n), dtype=torch.float64, device=dev)
        return tf
    allb = _compose_all(tf.blocks)
    Yd, _, Td = allb.device_parts(dev)
    Ap = ColMajor.empty(M.m, M.n, dev)
    Ap.view().copy_(M.view()[:, tf.perm_device(dev)])
    YtA = gemm_tn(Yd, Ap)
    tf._w_td = gemm_tn(Td, YtA).view().contiguous()
    return tf


def trqrcp(A, k: int, b: int = 32, p: int = 8, seed: int = 0, allow_large_k: bool = False,
           omega=None, _status=None) -> TruncatedFactorization:
    """Truncated RQRCP without trailing update (randomized.py:250-341)."""
    M, _ = _load(A)
    return _trqrcp_dev(M, k, b, p, seed, allow_large_k, omega, _status)


def _trqrcp_dev(M: ColMajor, k, b, p, seed, allow_large_k=False, omega=None, _status=None):
    """trqrcp on a validated device copy M, which the main path permutes in
    place (the reference's `work`, randomized.py:278, 299); the result's
    `_permuted_input` says whether it did."""
    m, n = M.m, M.n
    _check_block_args(m, n, k, b, p)
    if not allow_large_k and k > min(m, n) // 2:
        raise ValueError("trqrcp targets k <= min(m, n)/2; pass allow_large_k=True to override")
    dev = M.t.device
    if k == 0:
        return _empty(m, n, dev, truncated=True)
    ell = b + p
    if ell >= m:
        return _truncated_from_pivoted(_fallback_qrcp(M, k, b, True), M)
    if b > MAX_B or ell > MAX_ELL:   # wider than the fused driver: per-block loop (wide.py)
        from .wide import trqrcp_wide
        return trqrcp_wide(M, k, b, p, seed, _omega_T(omega, ell, m, seed, dev))
    L = _lib.lib()
    OmT = _omega_T(omega, ell, m, seed, dev)
    A0 = M  # permuted in place (the reference's `work`); the caller's A is untouched
    nblk = -(-k // b)
    Yg = ColMajor.empty(m, k, dev, zero=True)
    Wg = ColMajor.empty(k, n, dev, zero=True)
    Rg = ColMajor.empty(k, n, dev, zero=True)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    taus = torch.zeros(k, dtype=torch.float64, device=dev)
    Tb = torch.zeros((nblk, b * b), dtype=torch.float64, device=dev)
    st = status_new(dev)
    with _ws(L.sqr_trqrcp_workspace(m, n, k, b, p), dev) as ws:
        _lib.check(L.sqr_trqrcp(A0.ptr, A0.ld, m, n, k, b, p, seed & ((1 << 64) - 1),
                                OmT.ptr if OmT is not None else None, OmT.ld if OmT is not None else 0,
                                Yg.ptr, Yg.ld, Wg.ptr, Wg.ld, Rg.ptr, Rg.ld, ptr(perm), ptr(taus), ptr(Tb),
                                ptr(st), ptr(ws), ws.numel(), stream_handle()), "sqr_trqrcp")
    s = status_read(st)
    if _status is not None:
        _status.append(s)
    ach, nb = int(s["achieved"]), int(s["nblocks"])
    tf = TruncatedFactorization(m, n, None, None, None, ach, trqrcp_counters(m, n, b, ell, ach, nb))
    tf._Rd = _upper_rows(Rg, ach)
    tf._permd = perm
    tf._w_td = Wg.view()[:ach, :].contiguous()
    widths = [(J * b, min(b, ach - J * b)) for J in range(nb)]
    tf._blocks_fn = lambda: _packed_blocks(Yg, taus, Tb, b, widths, m)
    tf._Yg = Yg
    tf._permuted_input = True
    return tf


def tuxv(A, k: int, j_max: int = 1, b: int = 32, p: int = 8, seed: int = 0, refine_sigma: bool = False,
         allow_large_k: bool = False, omega=None) -> TuxvResult:
    """TRQRCP + QLP flip-flop passes (randomized.py:353-406)."""
    if j_max < 1:
        raise ValueError("j_max must be >= 1")
    # ONE validated device copy of A (one H2D for host input): TRQRCP permutes
    # it in place, after which the flip-flop products use (A P)(P^T V_k) = A V_k
    # and U^T (A P) = (U^T A) P on the permuted copy.
    M, _ = _load(A)
    tf = _trqrcp_dev(M, k, b, p, seed, allow_large_k, omega)
    m, n = M.m, M.n
    dev = M.t.device
    permuted = getattr(tf, "_permuted_input", False)
    L = _lib.lib()
    permd = tf.perm_device(dev)

    def a_times(Vk: ColMajor) -> ColMajor:            # A V_k  (m x kh)
        if permuted:                                   # P^T V_k for the permuted copy
            Vp = ColMajor.empty(Vk.m, Vk.n, dev)
            _lib.check(L.sqr_gather_rows(Vk.ptr, Vk.ld, Vk.m, Vk.n, permd.data_ptr(), Vp.ptr, Vp.ld,
                                         stream_handle()), "sqr_gather_rows")
            Vk = Vp
        return gemm_nn(M, Vk)

    def at_times(Uk: ColMajor) -> ColMajor:           # (U_k^T A)^T  (n x kh)
        Zt = gemm_tn(Uk, M)                            # kh x n  (= U^T A P on the permuted copy)
        Z = ColMajor.empty(n, Uk.n, dev)
        if permuted:                                   # (U^T A)^T = P (U^T A P)^T: scatter rows
            Ztt = _transpose(Zt)
            _lib.check(L.sqr_scatter_rows(Ztt.ptr, Ztt.ld, n, Uk.n, permd.data_ptr(), Z.ptr, Z.ld,
                                          stream_handle()), "sqr_scatter_rows")
        else:
            Z.view().copy_(Zt.view().T)
        return Z

    return _qlp(tf, m, n, b, j_max, refine_sigma, a_times, at_times, dev)


def _qlp(tf, m: int, n: int, b: int, j_max: int, refine_sigma: bool, a_times, at_times, dev) -> TuxvResult:
    """The QLP flip-flop of TUXV after its TRQRCP (randomized.py:367-406), with
    the two products of A supplied by the caller (single GPU: the permuted
    device copy; multi-GPU: local slabs + all-reduce / all-gather)."""
    L = _lib.lib()
    kh = tf.achieved_rank
    cnt = tf.counters
    if kh == 0:
        return TuxvResult(None, np.zeros((0, 0)), None, np.zeros(0), 0, cnt, m, n)
    # Z0 = R P^T; LQ of Z0 via QR of Z0^T (n x kh)
    # Z0^T = (R P^T)^T: row j of R^T goes to row perm[j] (scatter, no inverse)
    Rd = tf.R_device(dev)                                  # (kh, n) row-major = R^T column-major, ld n
    permd = tf.perm_device(dev)
    Z0t = ColMajor.empty(n, kh, dev)
    _lib.check(L.sqr_scatter_rows(Rd.data_ptr(), n, n, kh, permd.data_ptr(), Z0t.ptr, Z0t.ld, stream_handle()),
               "sqr_scatter_rows")
    vf = _qr_blocked_dev(Z0t, kh, b)
    cnt.merge(vf.counters)
    # the flip-flop passes use each factor as one composed block (QLP: U, V
    # of the result are the compositions, randomized.py:344-350, 396-406)
    v_blocks, u_blocks = vf._composed_fn(), []
    X = vf.R_device(dev)[:kh, :kh].T.contiguous()
    for j in range(1, j_max + 1):
        if j % 2 == 1:
            Z = a_times(_q_columns_dev(v_blocks, n, kh, dev))
            cnt.add_pass()
            cnt.add_blas3(m, n, kh)
            uf = _qr_blocked_dev(Z, kh, b)
            cnt.merge(uf.counters)
            u_blocks = uf._composed_fn()
            X = uf.R_device(dev)[:kh, :kh].contiguous()
        else:
            Z = at_times(_q_columns_dev(u_blocks, m, kh, dev))
            cnt.add_pass()
            cnt.add_blas3(kh, m, n)
            vf = _qr_blocked_dev(Z, kh, b)
            cnt.merge(vf.counters)
            v_blocks = vf._composed_fn()
            X = vf.R_device(dev)[:kh, :kh].T.contiguous()
    sig = torch.abs(torch.diagonal(X))
    if refine_sigma:                                   # randomized.py:402-403
        Xc = ColMajor.empty(kh, kh, dev)
        Xc.view().copy_(X)
        sig = _jacobi_svd_dev(Xc)[1]
    return TuxvResult(_compose_all(u_blocks), X, _compose_all(v_blocks), sig, kh, cnt, m, n)


# ------------------------------------------------------------ Jacobi SVD
_JACOBI_SWEEPS = 60


def _jacobi_svd_dev(M: ColMajor, want_u: bool = False):
    """(U, sigma, V) of the m x n device matrix M (m >= n), one-sided Jacobi
    on the device (sqr_jacobi_svd, jacobi.py:50-117); M is overwritten.
    U is None unless want_u."""
    m, n = M.m, M.n
    dev = M.t.device
    V = ColMajor.empty(n, n, dev)
    sig = torch.empty(n, dtype=torch.float64, device=dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().sqr_jacobi_svd(M.ptr, M.ld, m, n, V.ptr, V.ld, ptr(sig), ptr(order), _JACOBI_SWEEPS,
                                         ptr(info), stream_handle()), "sqr_jacobi_svd")
    if int(info[0].item()) < 0:
        raise np.linalg.LinAlgError("Jacobi sweeps did not converge")
    L = _lib.lib()
    sig = sig[order]
    Vs = ColMajor.empty(n, n, dev)
    _lib.check(L.sqr_copy_columns(V.ptr, V.ld, n, ptr(order), Vs.ptr, Vs.ld, None, n, stream_handle()), "sort V")
    if not want_u:
        return None, sig, Vs
    Ws = ColMajor.empty(m, n, dev)
    _lib.check(L.sqr_copy_columns(M.ptr, M.ld, m, ptr(order), Ws.ptr, Ws.ld, None, n, stream_handle()), "sort W")
    smax = float(sig[0])
    r = int(torch.count_nonzero(sig > smax * m * np.finfo(np.float64).eps))
    U = ColMajor.empty(m, n, dev, zero=True)
    if r:
        U.view()[:, :r] = Ws.view()[:, :r] / sig[:r]
    if r < n:   # orthonormal completion: columns r..n of the complete QR of U[:, :r] (jacobi.py:40-47)
        Ur = ColMajor.empty(m, r, dev)
        Ur.view().copy_(U.view()[:, :r])
        qf = _qr_blocked_dev(Ur, r, 32)
        U.view()[:, r:] = _q_columns_dev(qf.blocks, m, n, dev).view()[:, r:]
    return U, sig, Vs


def jacobi_svd(A):
    """Economy SVD (U, sigma, V), A = U diag(sigma) V^T, sigma descending, by
    one-sided Jacobi on the device (jacobi.py:50-117; same rotations, sweep
    rule, ordering and rank-deficient completion)."""
    M, _ = _load(A)
    m, n = M.m, M.n
    if min(m, n) > 4096:
        raise ValueError("jacobi_svd targets desk-scale matrices (min dim <= 4096)")
    if m < n:
        V, s, U = jacobi_svd(_transpose(M).view())
        return U, s, V
    if n == 0:
        return np.zeros((m, 0)), np.zeros(0), np.zeros((0, 0))
    if float(torch.linalg.norm(M.view())) == 0.0:
        return np.eye(m, n), np.zeros(n), np.eye(n)
    U, sig, V = _jacobi_svd_dev(M, want_u=True)
    return U.numpy(), sig.cpu().numpy(), V.numpy()

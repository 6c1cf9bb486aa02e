"""Out-of-bounds write guards (compute-sanitizer is closed on this GPU pool, see
DESIGN.md §7): every output of the C-ABI entry points is placed inside a
larger allocation whose surrounding bands hold NaN canaries (and, for
matrices, a leading dimension larger than the row count, whose padding rows
are canaries too).  After the call on awkward shapes (ragged sizes, one-
column panels, tall / wide, b = 1, l >= 144, n_t spanning several CTAs and
the cluster / grid-barrier paths), every canary must be untouched and every
result finite; the results are compared with the oracle where it is cheap.
"""
import numpy as np
import pytest

from conftest import gauss
from oracle import port as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2008_04447_b200 import _lib  # noqa: E402
from paper_2008_04447_b200._dev import stream_handle  # noqa: E402

DEV = torch.device("cuda", 0)
L = _lib.lib()
BAND = 4096  # canary elements before and after every buffer


class Guarded:
    """A column-major rows x cols fp64 matrix with leading dimension ld > rows,
    inside a buffer with NaN bands before / after and NaN padding rows."""

    def __init__(self, rows, cols, ld=None, data=None, dtype=torch.float64):
        self.rows, self.cols = rows, cols
        self.ld = ld if ld is not None else rows + 3
        self.dtype = dtype
        canary = float("nan") if dtype == torch.float64 else -7777
        self.buf = torch.full((2 * BAND + self.ld * max(cols, 1),), canary, dtype=dtype, device=DEV)
        self.body = self.buf[BAND:BAND + self.ld * max(cols, 1)].view(max(cols, 1), self.ld)
        self.canary = canary
        if data is not None:
            self.body[:cols, :rows] = torch.as_tensor(np.ascontiguousarray(np.asarray(data).T), device=DEV)
        elif dtype == torch.float64:
            self.body[:cols, :rows] = 0.0
        else:
            self.body[:cols, :rows] = 0

    @property
    def ptr(self):
        return self.body.data_ptr()

    def numpy(self):
        return self.body[:self.cols, :self.rows].cpu().numpy().T

    def intact(self):
        b = self.buf
        pads = [b[:BAND], b[BAND + self.ld * max(self.cols, 1):], self.body[:, self.rows:].reshape(-1)]
        for p in pads:
            if self.dtype == torch.float64:
                if not bool(torch.isnan(p).all()):
                    return False
            elif not bool((p == self.canary).all()):
                return False
        return True


def ws(nbytes):
    return torch.zeros(int(nbytes) + 4096, dtype=torch.uint8, device=DEV)


@pytest.mark.parametrize("m,n,k,b,p", [(97, 61, 61, 7, 3), (300, 257, 200, 1, 0), (40, 300, 33, 16, 8),
                                       (2000, 5000, 256, 128, 16), (1500, 4100, 300, 64, 80),
                                       (39000, 70, 70, 32, 8)])
def test_rqrcp_driver_writes_stay_in_bounds(m, n, k, b, p):
    if b + p > 144:
        pytest.skip("fused driver limit (wide blocks run wide.py on the same kernels)")
    A = gauss(m, n, m + n)
    Ag = Guarded(m, n, data=A)
    perm = Guarded(n, 1, ld=n, dtype=torch.int64)
    nblk = -(-k // b)
    taus = Guarded(k, 1, ld=k)
    T = Guarded(b * b, nblk, ld=b * b)
    st = torch.zeros(72, dtype=torch.uint8, device=DEV)
    OmT = Guarded(m, b + p, data=O.gauss_matrix(b + p, m, 0).T)
    w = ws(L.sqr_rqrcp_workspace(m, n, k, b, p))
    _lib.check(L.sqr_rqrcp(Ag.ptr, Ag.ld, m, n, k, b, p, 0, OmT.ptr, OmT.ld, 0, perm.ptr, taus.ptr, T.ptr,
                           st.data_ptr(), w.data_ptr(), w.numel(), stream_handle()))
    torch.cuda.synchronize()
    for g in (Ag, perm, taus, T, OmT):
        assert g.intact()
    ref = O.rqrcp(A, k, b=b, p=p, seed=0)
    assert np.array_equal(perm.numpy()[:, 0], ref.perm)
    R = np.triu(Ag.numpy()[:ref.achieved_rank])
    assert np.abs(R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()


@pytest.mark.parametrize("m,n,k,b,p", [(97, 61, 20, 7, 3), (1200, 900, 96, 32, 8), (5000, 300, 128, 128, 8)])
def test_trqrcp_driver_writes_stay_in_bounds(m, n, k, b, p):
    A = gauss(m, n, 3 * m + n)
    Ag = Guarded(m, n, data=A)
    Yg, Wg, Rg = Guarded(m, k), Guarded(k, n), Guarded(k, n)
    perm = Guarded(n, 1, ld=n, dtype=torch.int64)
    taus = Guarded(k, 1, ld=k)
    T = Guarded(b * b, -(-k // b), ld=b * b)
    st = torch.zeros(72, dtype=torch.uint8, device=DEV)
    OmT = Guarded(m, b + p, data=O.gauss_matrix(b + p, m, 0).T)
    w = ws(L.sqr_trqrcp_workspace(m, n, k, b, p))
    _lib.check(L.sqr_trqrcp(Ag.ptr, Ag.ld, m, n, k, b, p, 0, OmT.ptr, OmT.ld, Yg.ptr, Yg.ld, Wg.ptr, Wg.ld,
                            Rg.ptr, Rg.ld, perm.ptr, taus.ptr, T.ptr, st.data_ptr(), w.data_ptr(), w.numel(),
                            stream_handle()))
    torch.cuda.synchronize()
    for g in (Ag, Yg, Wg, Rg, perm, taus, T, OmT):
        assert g.intact()
    ref = O.trqrcp(A, k, b=b, p=p, seed=0, allow_large_k=True)
    assert np.array_equal(perm.numpy()[:, 0], ref.perm)
    assert np.abs(Wg.numpy()[:ref.achieved_rank] - ref.w_t).max() <= 1e-10 * np.abs(ref.w_t).max()


@pytest.mark.parametrize("mr,w", [(1, 1), (37, 5), (257, 33), (9000, 128), (38000, 64), (80000, 16)])
def test_panel_writes_stay_in_bounds(mr, w):
    P = gauss(mr, w, mr + w)
    Pg = Guarded(mr, w, data=P)
    Y = Guarded(mr, w)
    taus = Guarded(w, 1, ld=w)
    st = torch.zeros(72, dtype=torch.uint8, device=DEV)
    wsb = ws(L.sqr_block_workspace(mr, 0, w))
    _lib.check(L.sqr_panel_factor(Pg.ptr, Pg.ld, mr, w, Y.ptr, Y.ld, taus.ptr, 1, st.data_ptr(), wsb.data_ptr(),
                                  wsb.numel(), stream_handle()))
    torch.cuda.synchronize()
    for g in (Pg, Y, taus):
        assert g.intact()
    work = np.asfortranarray(P.copy())
    Yp, tp, bh = O.panel_factor(work, 0, min(w, mr))
    got = Pg.numpy()
    assert np.abs(np.triu(got[:w]) - np.triu(work[:w])).max() <= 1e-12 * max(np.abs(work).max(), 1.0)


@pytest.mark.parametrize("ell,nt,bb", [(1, 1, 1), (9, 300, 9), (136, 4096, 128), (136, 4097, 128),
                                       (150, 900, 100), (40, 40000, 32)])
def test_sample_qrcp_writes_stay_in_bounds(ell, nt, bb):
    B = gauss(ell, nt, ell * nt)
    Bg = Guarded(ell, nt, data=B)
    Bf = Guarded(ell, nt)
    lperm = Guarded(nt, 1, ld=nt, dtype=torch.int64)
    moves = Guarded(4 * bb + 8, 1, ld=4 * bb + 8, dtype=torch.int32)
    taus = Guarded(bb, 1, ld=bb)
    st = torch.zeros(72, dtype=torch.uint8, device=DEV)
    _lib.check(L.sqr_sample_qrcp(Bg.ptr, Bg.ld, ell, nt, bb, Bf.ptr, Bf.ld, lperm.ptr, moves.ptr, taus.ptr, 1,
                                 st.data_ptr(), stream_handle()))
    torch.cuda.synchronize()
    for g in (Bg, Bf, lperm, moves, taus):
        assert g.intact()
    ref = O.sample_pivots(B, bb)
    assert np.array_equal(lperm.numpy()[:ref.achieved, 0], ref.local_perm[:ref.achieved])


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (144, 77, 3001), (33, 4100, 129), (128, 32640, 512)])
def test_gemms_write_stay_in_bounds(M, N, K):
    rng = np.random.default_rng(M + N + K)
    X = rng.standard_normal((K, M))
    C = rng.standard_normal((K, N))
    Xg, Cg, Dg = Guarded(K, M, data=X), Guarded(K, N, data=C), Guarded(M, N)
    w = ws(200 << 20)
    _lib.check(L.sqr_gemm_tn(M, N, K, 1.0, Xg.ptr, Xg.ld, Cg.ptr, Cg.ld, 0.0, None, 0, Dg.ptr, Dg.ld, w.data_ptr(),
                             w.numel(), stream_handle()))
    Y = rng.standard_normal((K, N))
    Xn = rng.standard_normal((M, K))
    Xng, Yg, En = Guarded(M, K, data=Xn), Guarded(K, N, data=Y), Guarded(M, N)
    _lib.check(L.sqr_gemm_nn(M, N, K, 1.0, Xng.ptr, Xng.ld, Yg.ptr, Yg.ld, 0.0, None, 0, En.ptr, En.ld,
                             stream_handle()))
    torch.cuda.synchronize()
    for g in (Xg, Cg, Dg, Xng, Yg, En):
        assert g.intact()
    assert np.abs(Dg.numpy() - X.T @ C).max() <= 1e-12 * np.abs(X.T @ C).max()
    assert np.abs(En.numpy() - Xn @ Y).max() <= 1e-12 * np.abs(Xn @ Y).max()

"""Kernel-level parity of libsqr against the CPU oracle / NumPy (needs a B200).

Each test calls one C-ABI entry point through ctypes on torch-owned device
memory and compares with the oracle restatement of the reference routine it
implements (oracle/port.py), at sizes the oracle finishes in seconds.
"""
import numpy as np
import pytest

from conftest import gauss, load_golden
from oracle import port as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2008_04447_b200 import _lib  # noqa: E402
from paper_2008_04447_b200._dev import ColMajor, status_new, status_read, stream_handle, upload  # noqa: E402

DEV = torch.device("cuda", 0)
L = _lib.lib()


def ws(nbytes):
    return torch.zeros(int(nbytes) + 4096, dtype=torch.uint8, device=DEV)


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)) if b.size else 0.0


# ------------------------------------------------------------------ Omega
@pytest.mark.parametrize("rows,cols,seed,offset", [(40, 1000, 0, 0), (72, 333, 7, 5), (136, 4097, 2**63 + 17, 11)])
def test_gaussian_matches_stream(rows, cols, seed, offset):
    out = ColMajor.empty(rows, cols, DEV)
    _lib.check(L.sqr_gaussian(out.ptr, out.ld, rows, cols, seed, offset, 0, stream_handle()))
    got = out.numpy()
    want = O.gauss_matrix(rows, cols, seed, offset)
    ulp = np.abs(got - want) / np.spacing(np.abs(want))
    assert ulp.max() <= 4, ulp.max()            # log/sin/cos: CUDA libm vs NumPy
    assert (got == want).mean() >= 0.8           # most entries bit-identical (86% measured)
    outT = ColMajor.empty(cols, rows, DEV)
    _lib.check(L.sqr_gaussian(outT.ptr, outT.ld, rows, cols, seed, offset, 1, stream_handle()))
    assert np.array_equal(outT.numpy(), got.T)


# ------------------------------------------------------------------ GEMMs
# the last three are wide enough (>= 148 tiles of 64 columns) for the two-launch schedule of long sweeps
# (whole waves at one split, the remaining tiles at a higher split; csrc/gemm_tma.cu)
@pytest.mark.parametrize("M,N,K,off", [(40, 1000, 1000, 0), (136, 700, 5000, 0), (128, 300, 70001, 0),
                                       (33, 129, 17, 1), (144, 1, 3, 0), (7, 513, 4096, 1), (128, 128, 32768, 0),
                                       (128, 12000, 8192, 0), (64, 20224, 5000, 0), (32, 9500, 20000, 0)])
def test_gemm_tn(M, N, K, off):
    rng = np.random.default_rng(M * N + K)
    X = rng.standard_normal((K + off, M))
    C = rng.standard_normal((K + off, N))
    E = rng.standard_normal((M, N))
    Xd, Cd, Ed = upload(X, DEV), upload(C, DEV), upload(E, DEV)
    D = ColMajor.empty(M, N, DEV)
    w = ws(200 << 20)
    _lib.check(L.sqr_gemm_tn(M, N, K, 0.5, Xd.col_ptr(off, 0), Xd.ld, Cd.col_ptr(off, 0), Cd.ld, -2.0, Ed.ptr, Ed.ld,
                             D.ptr, D.ld, w.data_ptr(), w.numel(), stream_handle()))
    want = 0.5 * X[off:].T @ C[off:] - 2.0 * E
    assert relerr(D.numpy(), want) <= 1e-13
    # deterministic: a second launch is bitwise identical
    D2 = ColMajor.empty(M, N, DEV)
    _lib.check(L.sqr_gemm_tn(M, N, K, 0.5, Xd.col_ptr(off, 0), Xd.ld, Cd.col_ptr(off, 0), Cd.ld, -2.0, Ed.ptr, Ed.ld,
                             D2.ptr, D2.ld, w.data_ptr(), w.numel(), stream_handle()))
    assert torch.equal(D.view(), D2.view())


@pytest.mark.parametrize("M,N,K,off", [(1000, 1000, 32, 0), (4097, 300, 128, 0), (513, 77, 3, 1), (20000, 100, 20000, 0),
                                       (100, 4000, 232, 1), (128, 20000, 128, 0), (77, 19001, 256, 1)])
def test_gemm_nn(M, N, K, off):
    rng = np.random.default_rng(M + N * K)
    X = rng.standard_normal((M + off, K))
    Y = rng.standard_normal((K + off, N))
    E = rng.standard_normal((M, N))
    Xd, Yd, Ed = upload(X, DEV), upload(Y, DEV), upload(E, DEV)
    _lib.check(L.sqr_gemm_nn(M, N, K, -1.0, Xd.col_ptr(off, 0), Xd.ld, Yd.col_ptr(off, 0), Yd.ld, 1.0, Ed.ptr, Ed.ld,
                             Ed.ptr, Ed.ld, stream_handle()))
    want = E - X[off:] @ Y[off:]
    assert relerr(Ed.numpy(), want) <= 1e-13


# ------------------------------------------------------------ sample QRCP
# shapes cover the thread-per-column kernel (nt <= 148*256, ell <= 144: odd ell,
# ell below / at the 48 register rows, ell = 144) and the smem/L2 kernel
# (nt > 37888 or ell > 144)
@pytest.mark.parametrize("ell,nt,bb,seed", [(40, 1000, 32, 1), (12, 40, 6, 5), (136, 6000, 128, 2), (72, 2000, 64, 3),
                                            (40, 20000, 32, 4), (9, 9, 9, 6), (137, 3000, 128, 7), (144, 700, 128, 8),
                                            (47, 257, 40, 9), (48, 513, 48, 12), (40, 40000, 32, 10),
                                            (150, 600, 100, 11)])
def test_sample_qrcp_matches_oracle(ell, nt, bb, seed):
    B = gauss(ell, nt, seed)
    st_ref = O.sample_pivots(B, bb)
    Bd = upload(B, DEV)
    Bf = ColMajor.empty(ell, nt, DEV)
    lperm = torch.empty(nt, dtype=torch.int64, device=DEV)
    moves = torch.empty(4 * bb + 8, dtype=torch.int32, device=DEV)
    taus = torch.zeros(bb, dtype=torch.float64, device=DEV)
    st = status_new(DEV)
    _lib.check(L.sqr_sample_qrcp(Bd.ptr, Bd.ld, ell, nt, bb, Bf.ptr, Bf.ld, lperm.data_ptr(), moves.data_ptr(),
                                 taus.data_ptr(), 1, st.data_ptr(), stream_handle()))
    s = status_read(st)
    assert int(s["sample_achieved"]) == st_ref.achieved
    assert np.array_equal(lperm.cpu().numpy(), st_ref.local_perm)
    a = st_ref.achieved
    got = Bf.numpy()
    assert relerr(np.triu(got[:a, :a]), st_ref.S11) <= 1e-12
    assert relerr(got[:a, a:], st_ref.S12) <= 1e-12
    assert relerr(got[a:, a:], st_ref.S22) <= 1e-11
    assert relerr(taus.cpu().numpy()[:a], st_ref.u_block.tau) <= 1e-12
    mv = moves.cpu().numpy()[: 2 * int(s["nmoves"])].reshape(-1, 2)
    mv = mv[mv[:, 0] >= 0]  # dst = -1 marks an unused slot
    assert np.unique(mv[:, 0]).size == mv.shape[0] and np.unique(mv[:, 1]).size == mv.shape[0]
    lp = np.arange(nt)
    lp[mv[:, 0]] = mv[:, 1]
    assert np.array_equal(lp, st_ref.local_perm)


def test_sample_qrcp_ties_and_exhaustion():
    g = np.zeros((2, 3), order="F")
    g[:, 0] = (3.0, 4.0)
    g[:, 2] = (4.0, 3.0)
    g[:, 1] = (0.1, 0.0)
    for B, bb in [(g, 2), (np.zeros((4, 6), order="F"), 2)]:
        ref = O.sample_pivots(B, bb)
        Bd = upload(B, DEV)
        Bf = ColMajor.empty(*B.shape, DEV)
        lperm = torch.empty(B.shape[1], dtype=torch.int64, device=DEV)
        moves = torch.empty(64, dtype=torch.int32, device=DEV)
        taus = torch.zeros(8, dtype=torch.float64, device=DEV)
        st = status_new(DEV)
        _lib.check(L.sqr_sample_qrcp(Bd.ptr, Bd.ld, B.shape[0], B.shape[1], bb, Bf.ptr, Bf.ld, lperm.data_ptr(),
                                     moves.data_ptr(), taus.data_ptr(), 1, st.data_ptr(), stream_handle()))
        s = status_read(st)
        assert int(s["sample_achieved"]) == ref.achieved
        if ref.achieved:
            assert np.array_equal(lperm.cpu().numpy()[: ref.achieved], ref.local_perm[: ref.achieved])
    B = np.zeros((4, 6), order="F")
    B[:, 2] = 1.0
    ref = O.sample_pivots(B, 3)
    assert ref.achieved == 1


# --------------------------------------------------------- sample update
def _sample_then_update(B, bb, R11, R12, entry="sqr_sample_update"):
    """sqr_sample_qrcp on B, then Bnext = [S12 - S11 R11^-1 R12; S22] through the ABI."""
    ell, ntot = B.shape
    Bd = upload(B, DEV)
    Bf = ColMajor.empty(ell, ntot, DEV)
    lperm = torch.empty(ntot, dtype=torch.int64, device=DEV)
    moves = torch.empty(4 * bb + 8, dtype=torch.int32, device=DEV)
    taus = torch.zeros(bb, dtype=torch.float64, device=DEV)
    st = status_new(DEV)
    _lib.check(L.sqr_sample_qrcp(Bd.ptr, Bd.ld, ell, ntot, bb, Bf.ptr, Bf.ld, lperm.data_ptr(), moves.data_ptr(),
                                 taus.data_ptr(), 1, st.data_ptr(), stream_handle()))
    R = upload(np.hstack([R11, R12]), DEV)
    nt = R12.shape[1]
    Bn = ColMajor.empty(ell, nt, DEV)
    if entry == "sqr_sample_update":
        _lib.check(L.sqr_sample_update(Bf.ptr, Bf.ld, ell, R.ptr, R.ld, nt, Bn.ptr, Bn.ld, st.data_ptr(),
                                       stream_handle()))
    elif entry == "sqr_sample_update_b":
        mbuf = torch.zeros(bb * bb, dtype=torch.float64, device=DEV)
        _lib.check(L.sqr_sample_update_b(Bf.ptr, Bf.ld, ell, R.ptr, R.ld, nt, bb, Bn.ptr, Bn.ld, st.data_ptr(),
                                         mbuf.data_ptr(), stream_handle()))
    else:  # prep + apply halves
        mbuf = torch.zeros(bb * bb, dtype=torch.float64, device=DEV)
        _lib.check(L.sqr_sample_update_prep(Bf.ptr, Bf.ld, R.ptr, R.ld, bb, mbuf.data_ptr(), st.data_ptr(),
                                            stream_handle()))
        _lib.check(L.sqr_sample_update_apply(Bf.ptr, Bf.ld, ell, R.ptr, R.ld, nt, bb, Bn.ptr, Bn.ld, st.data_ptr(),
                                             mbuf.data_ptr(), stream_handle()))
    return Bn.numpy(), status_read(st)


@pytest.mark.parametrize("entry", ["sqr_sample_update", "sqr_sample_update_b", "prep_apply"])
def test_sample_update_golden(entry):
    """sketch.py:132-149 against the REAL reference's sample_update output
    (tests/golden/sample.npz: s_next)."""
    g = load_golden("sample")
    got, s = _sample_then_update(g["sB"], 6, g["s_R11"], g["s_R12"], entry)
    assert int(s["stop"]) == 0
    assert relerr(got, g["s_next"]) <= 1e-12


@pytest.mark.parametrize("ell,ntot,bb,seed", [(40, 1000, 32, 1), (136, 6000, 128, 2), (72, 2001, 64, 3), (9, 30, 1, 4)])
def test_sample_update_matches_oracle(ell, ntot, bb, seed):
    B = gauss(ell, ntot, seed)
    ref = O.sample_pivots(B, bb)
    R11 = np.triu(gauss(bb, bb, seed + 100)) + 3 * np.eye(bb)
    R12 = gauss(bb, ntot - bb, seed + 200)
    want = O.sample_refresh(ref, R11, R12)
    for entry in ("sqr_sample_update", "sqr_sample_update_b"):
        got, s = _sample_then_update(B, bb, R11, R12, entry)
        assert int(s["stop"]) == 0
        assert relerr(got, want) <= 1e-11


def test_sample_update_singular_guard():
    """_diag_ok (randomized.py:133-135): min |R11_ii| <= 2^-52 |R11_00| stops the
    loop (reason r11_singular) instead of solving, as the reference breaks."""
    B = gauss(12, 40, 5)
    R11 = np.triu(gauss(6, 6, 6)) + 4 * np.eye(6)
    R11[3, 3] = 2.0 ** -60 * abs(R11[0, 0])
    with pytest.raises(np.linalg.LinAlgError):
        O.sample_refresh(O.sample_pivots(B, 6), R11, gauss(6, 34, 7))
    _, s = _sample_then_update(B, 6, R11, gauss(6, 34, 7))
    assert int(s["stop"]) == 1 and _lib.STOP_REASONS[int(s["reason"])] == "r11_singular"


# ----------------------------------------------------------------- panel
@pytest.mark.parametrize("mr,w,seed", [(1000, 32, 1), (5000, 64, 2), (32768, 128, 3), (100000, 64, 4), (257, 13, 5)])
def test_panel_matches_oracle(mr, w, seed):
    P = gauss(mr, w, seed)
    work = P.copy(order="F")
    Yref, tref, done = O.panel_factor(work, 0, w)
    Pd = upload(P, DEV)
    Y = ColMajor.empty(mr, w, DEV)
    taus = torch.zeros(w, dtype=torch.float64, device=DEV)
    T = ColMajor.empty(w, w, DEV)
    st = status_new(DEV)
    _lib.check(L.sqr_panel_qr(Pd.ptr, Pd.ld, mr, w, Y.ptr, Y.ld, taus.data_ptr(), T.ptr, T.ld, 1, st.data_ptr(),
                              stream_handle()))
    s = status_read(st)
    assert int(s["bhat"]) == done == w
    assert relerr(Pd.numpy(), work) <= 1e-11
    assert relerr(Y.numpy(), Yref) <= 1e-11
    assert relerr(taus.cpu().numpy(), tref) <= 1e-12
    assert relerr(T.numpy(), O.t_factor(Yref, tref)) <= 1e-11


def test_panel_zero_column_stops_like_reference():
    P = gauss(300, 24, 9)
    P[:, 5] = P[:, 2] * 0.0  # exactly zero column -> beta == 0 at t = 5
    work = P.copy(order="F")
    Yref, tref, done = O.panel_factor(work, 0, 24)
    assert done == 5
    Pd = upload(P, DEV)
    Y = ColMajor.empty(300, 24, DEV)
    taus = torch.zeros(24, dtype=torch.float64, device=DEV)
    st = status_new(DEV)
    _lib.check(L.sqr_panel_qr(Pd.ptr, Pd.ld, 300, 24, Y.ptr, Y.ld, taus.data_ptr(), None, 0, 1, st.data_ptr(),
                              stream_handle()))
    s = status_read(st)
    assert int(s["bhat"]) == 5
    assert relerr(Pd.numpy(), work) <= 1e-11
    assert relerr(Y.numpy()[:, :5], Yref) <= 1e-11
    assert np.all(Y.numpy()[:, 5:] == 0.0)


# ------------------------------------------------ whole-panel factor (C ABI)
def _panel_factor_dev(P, w, stop_at_zero=1):
    mr = P.shape[0]
    Pd = upload(P, DEV)
    Y = ColMajor.empty(mr, w, DEV)
    taus = torch.zeros(w, dtype=torch.float64, device=DEV)
    st = status_new(DEV)
    ws = torch.zeros(int(L.sqr_block_workspace(mr, w, w)), dtype=torch.uint8, device=DEV)
    _lib.check(L.sqr_panel_factor(Pd.ptr, Pd.ld, mr, w, Y.ptr, Y.ld, taus.data_ptr(), stop_at_zero, st.data_ptr(),
                                  ws.data_ptr(), ws.numel(), stream_handle()))
    return Pd.numpy(), Y.numpy(), taus.cpu().numpy(), status_read(st)


# single-launch block kernel (mr <= 148*256) and the leaf + GEMM path beyond it
@pytest.mark.parametrize("mr,w,seed", [(1000, 32, 1), (5000, 100, 2), (32768, 128, 3), (37888, 128, 4),
                                       (40000, 64, 5), (257, 13, 6), (300, 33, 7), (64, 64, 8)])
def test_panel_factor_matches_oracle(mr, w, seed):
    P = gauss(mr, w, seed)
    work = P.copy(order="F")
    Yref, tref, done = O.panel_factor(work, 0, w)
    Pg, Yg, tg, s = _panel_factor_dev(P, w)
    assert int(s["bhat"]) == done == w
    assert relerr(Pg, work) <= 1e-11
    assert relerr(Yg, Yref) <= 1e-11
    assert relerr(tg, tref) <= 1e-12


@pytest.mark.parametrize("mr,w,zc", [(300, 24, 5), (2000, 100, 40), (2000, 100, 0), (50000, 64, 37)])
def test_panel_factor_zero_column(mr, w, zc):
    P = gauss(mr, w, 9)
    P[:, zc] = 0.0  # exactly zero column: beta == 0 at step zc
    work = P.copy(order="F")
    Yref, tref, done = O.panel_factor(work, 0, w)
    assert done == zc
    Pg, Yg, tg, s = _panel_factor_dev(P, w)
    assert int(s["bhat"]) == zc
    assert relerr(Pg, work) <= 1e-11
    if zc:
        assert relerr(Yg[:, :zc], Yref) <= 1e-11
        assert relerr(tg[:zc], tref[:zc]) <= 1e-12
    assert np.all(Yg[:, zc:] == 0.0) and np.all(tg[zc:] == 0.0)
    if zc == 0:
        assert int(s["stop"]) == 1 and int(s["reason"]) == 4


@pytest.mark.parametrize("M,N,K,off", [(20000, 100, 20000, 0), (3000, 40, 9000, 1), (777, 130, 4100, 0)])
def test_gemm_nn_split_k(M, N, K, off):
    """sqr_gemm_nn_ws: skinny long-K products split K across CTAs (TUXV's
    A V_k); the fixed-order reduction is bitwise reproducible."""
    rng = np.random.default_rng(M + 7 * N + K)
    X = rng.standard_normal((M + off, K))
    Y = rng.standard_normal((K + off, N))
    E = rng.standard_normal((M, N))
    Xd, Yd, Ed = upload(X, DEV), upload(Y, DEV), upload(E, DEV)
    w = ws(16 * M * N * 8)
    outs = []
    for _ in range(2):
        D = ColMajor.empty(M, N, DEV)
        _lib.check(L.sqr_gemm_nn_ws(M, N, K, 0.5, Xd.col_ptr(off, 0), Xd.ld, Yd.col_ptr(off, 0), Yd.ld, -1.0, Ed.ptr,
                                    Ed.ld, D.ptr, D.ld, w.data_ptr(), w.numel(), stream_handle()))
        outs.append(D)
    want = 0.5 * X[off:] @ Y[off:] - E
    assert relerr(outs[0].numpy(), want) <= 1e-13
    assert torch.equal(outs[0].view(), outs[1].view())


# ------------------------------------------------- TMA vs cp.async GEMM paths
@pytest.mark.parametrize("kind,M,N,K", [("tn", 128, 1000, 5000), ("tn", 64, 777, 333), ("tn", 100, 300, 70001),
                                        ("nn", 1000, 1000, 256), ("nn", 4097, 300, 128), ("nn", 513, 129, 17)])
def test_tma_gemm_bitwise_equals_cp_async(kind, M, N, K, monkeypatch):
    """The TMA-staged warp-specialised GEMMs (csrc/gemm_tma.cu) accumulate in the
    same k order as the cp.async kernels: bitwise equal results (SQR_NO_TMA is
    read per call)."""
    rng = np.random.default_rng(M + N + K)
    E = upload(rng.standard_normal((M, N)), DEV)
    w = ws(400 << 20)
    if kind == "tn":
        X, C = upload(rng.standard_normal((K, M)), DEV), upload(rng.standard_normal((K, N)), DEV)
        call = lambda D: L.sqr_gemm_tn(M, N, K, 0.5, X.ptr, X.ld, C.ptr, C.ld, -2.0, E.ptr, E.ld, D.ptr, D.ld,
                                       w.data_ptr(), w.numel(), stream_handle())
    else:
        X, Y = upload(rng.standard_normal((M, K)), DEV), upload(rng.standard_normal((K, N)), DEV)
        call = lambda D: L.sqr_gemm_nn(M, N, K, 0.5, X.ptr, X.ld, Y.ptr, Y.ld, -2.0, E.ptr, E.ld, D.ptr, D.ld,
                                       stream_handle())
    out = []
    for off in (None, "1"):
        if off:
            monkeypatch.setenv("SQR_NO_TMA", off)
        else:
            monkeypatch.delenv("SQR_NO_TMA", raising=False)
        D = ColMajor.empty(M, N, DEV)
        _lib.check(call(D))
        out.append(D.numpy())
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("M,N,K,beta", [(1000, 1000, 256, 1.0), (4096, 300, 128, -0.5), (513, 129, 17, 1.0),
                                        (128, 5000, 128, 1.0)])
def test_gemm_nn_unit_alpha(M, N, K, beta):
    """alpha = 1, the trailing updates' form C + beta... (E in place of D)."""
    rng = np.random.default_rng(M * 7 + N + K)
    X, Y, E = rng.standard_normal((M, K)), rng.standard_normal((K, N)), rng.standard_normal((M, N))
    Xd, Yd, Ed = upload(X, DEV), upload(Y, DEV), upload(E, DEV)
    _lib.check(L.sqr_gemm_nn(M, N, K, 1.0, Xd.ptr, Xd.ld, Yd.ptr, Yd.ld, beta, Ed.ptr, Ed.ld, Ed.ptr, Ed.ld,
                             stream_handle()))
    want = X @ Y + beta * E
    assert relerr(Ed.numpy(), want) <= 1e-13

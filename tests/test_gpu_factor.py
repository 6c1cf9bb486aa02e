"""Driver-level parity: paper_2008_04447_b200 (libsqr on a B200) vs the CPU
oracle and the reference's golden fixtures.

Bars (north star): identical permutation; ||AP - QR||/||A|| <= 1e-12;
||Q^T Q - I||_max <= 1e-12; |R_jj| within 1e-10 relative per entry (normwise
|dR_jj|/|R_11| for the decaying spectra factored to full rank); identical
counters; truncation errors within 1e-10 relative of the oracle's.
"""
import numpy as np
import pytest

from conftest import gauss, golden_kwargs, load_golden
from oracle import port as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2008_04447_b200 as G  # noqa: E402


def counters_of(pf):
    c = pf.counters
    return [c.trailing_passes, c.blas2_volume, c.blas3_volume]


def first_mismatch(p1, p2):
    d = np.nonzero(np.asarray(p1) != np.asarray(p2))[0]
    return int(d[0]) if d.size else None


def check_against(pf, ref, A, rdiag_tol=1e-10, normwise=False, noise=1e-10):
    """Same pivots, except a documented near-tie: pivots chosen among columns
    already at the noise floor (oracle |R_jj| <= noise * |R_00|) may differ
    because rounding alone orders them."""
    assert pf.achieved_rank == ref.achieved_rank
    j = first_mismatch(pf.perm, ref.perm)
    if j is not None:
        dr = np.abs(ref.r_diag)
        assert j < dr.size and dr[j] <= noise * dr[0], f"pivot mismatch at {j} above the noise floor"
        assert np.abs(pf.r_diag[j:]).max() <= noise * dr[0]
        assert np.array_equal(pf.perm[:j], ref.perm[:j])
        return
    assert counters_of(pf) == [ref.counters.trailing_passes, ref.counters.blas2_volume, ref.counters.blas3_volume]
    r = pf.achieved_rank
    if r:
        d, dr = np.abs(pf.r_diag), np.abs(ref.r_diag)
        if normwise:
            assert np.abs(d - dr).max() <= rdiag_tol * dr[0]
        else:
            assert np.all(np.abs(d - dr) <= rdiag_tol * dr)
        scale = max(np.abs(ref.R).max(), 1e-300)
        assert np.abs(pf.R - ref.R).max() <= 1e-10 * scale
    assert len(pf.blocks) == len(ref.blocks)
    for b1, b2 in zip(pf.blocks, ref.blocks):
        assert b1.offset == b2.offset and b1.width == b2.width


RANDOMIZED = ["r_small", "r_ragged", "r_tall", "r_wide", "r_short", "r_rankdef", "r_zero", "r_diag64", "r_kahan",
              "rs_small", "ss_small"]


@pytest.mark.parametrize("name", RANDOMIZED)
def test_randomized_vs_golden_and_oracle(name):
    g = load_golden(name)
    kw = golden_kwargs(g)
    fn = {"r": G.rqrcp, "rs": G.rsrqrcp, "ss": G.ssrqrcp}[name.split("_")[0]]
    ofn = {"r": O.rqrcp, "rs": O.rsrqrcp, "ss": O.ssrqrcp}[name.split("_")[0]]
    A = g["A"]
    extra = {} if name.startswith("rs") else {"omega": "host"}
    pf = fn(A, **kw, **extra)
    ref = ofn(A, **kw)
    check_against(pf, ref, A, normwise=name in ("r_kahan", "r_rankdef"))
    j = first_mismatch(pf.perm, g["perm"])
    assert j is None or np.abs(g["rdiag"][j]) <= 1e-10 * np.abs(g["rdiag"][0])
    if pf.achieved_rank:
        assert pf.rel_residual(A) <= max(1e-12, 10 * float(g["rel_residual"]))
        Q = pf.q_columns()
        assert np.abs(Q.T @ Q - np.eye(Q.shape[1])).max() <= 1e-12


@pytest.mark.parametrize("name", ["t_small", "t_decay", "t_short", "t_large_k"])
def test_trqrcp_vs_golden_and_oracle(name):
    g = load_golden(name)
    kw = golden_kwargs(g)
    kw["allow_large_k"] = bool(kw.get("allow_large_k", 0))
    A = g["A"]
    tf = G.trqrcp(A, **kw, omega="host")
    ref = O.trqrcp(A, **kw)
    check_against(tf, ref, A)
    scale = max(np.abs(ref.w_t).max(), 1e-300)
    assert np.abs(tf.w_t - ref.w_t).max() <= 1e-10 * scale
    k = tf.achieved_rank
    assert abs(tf.rel_residual(A, k) - ref.rel_residual(A, k)) <= 1e-10 * ref.rel_residual(A, k)


def test_trqrcp_equals_rqrcp_on_device():
    for seed in range(3):
        A = gauss(100, 80, seed + 30)
        tf = G.trqrcp(A, 24, b=8, p=8, seed=seed)
        full = G.rqrcp(A, 24, b=8, p=8, seed=seed)
        assert np.array_equal(tf.perm[:24], full.perm[:24])
        assert np.abs(tf.R[:24, :] - full.R[:24, :]).max() <= 1e-10


@pytest.mark.parametrize("name", ["x_small", "x_flip2", "x_refine"])
def test_tuxv_vs_golden(name):
    g = load_golden(name)
    kw = golden_kwargs(g)
    if "refine_sigma" in kw:
        kw["refine_sigma"] = bool(kw["refine_sigma"])
    A = g["A"]
    res = G.tuxv(A, **kw, omega="host")
    assert res.achieved_rank == int(g["achieved"])
    scale = np.abs(g["recon"]).max()
    assert np.abs(res.reconstruct() - g["recon"]).max() <= 1e-9 * scale
    assert np.abs(np.abs(res.sigma_est) - np.abs(g["sigma_est"])).max() <= 1e-10 * np.abs(g["sigma_est"]).max()
    assert [res.counters.trailing_passes, res.counters.blas2_volume, res.counters.blas3_volume] == g["counters"].tolist()
    U, V = res.u_columns(), res.v_columns()
    k = res.achieved_rank
    assert np.abs(U.T @ U - np.eye(k)).max() <= 1e-12
    assert np.abs(V.T @ V - np.eye(k)).max() <= 1e-12


def test_deterministic_qr_routines():
    g = load_golden("qrcp")
    A = g["qA"]
    for fn, ofn, pre in [(lambda a: G.qrcp_blas2(a), O.qrcp_blas2, "blas2_"),
                         (lambda a: G.qrcp_blocked(a, b=8), lambda a: O.qrcp_blocked(a, b=8), "blocked_"),
                         (lambda a: G.qr_blocked(a, b=8), lambda a: O.qr_blocked(a, b=8), "qrb_")]:
        pf, ref = fn(A), ofn(A)
        check_against(pf, ref, A)
        assert np.array_equal(pf.perm, g[pre + "perm"])
    assert G.qrcp_blas2(np.diag([1.0, 2.0, 3.0])).perm.tolist() == [2, 1, 0]
    assert G.qrcp_blas2(np.eye(4)).perm.tolist() == [0, 1, 2, 3]
    assert G.qrcp_blocked(np.diag(np.arange(1.0, 9.0)), b=4).perm.tolist() == list(range(7, -1, -1))


def test_config1_device_omega():
    """C1 (BASELINE configs[0]) with the DEFAULT device-generated Omega: the
    oracle is fed the device's own Omega, so pivots must agree exactly."""
    g = load_golden("c1")
    A = O.gauss_matrix(1000, 1000, 1)
    pf = G.rqrcp(A, 1000, b=32, p=8, seed=0)
    om = G.device_giid(40, 1000, 0).cpu().numpy()
    ref = O.rqrcp(A, 1000, b=32, p=8, seed=0, omega=om)
    check_against(pf, ref, A)
    assert counters_of(pf) == g["counters"].tolist()
    # and against the reference itself (host Omega in the reference): same pivots
    assert np.array_equal(pf.perm, g["perm"])
    assert pf.rel_residual(A) <= 1e-12


def test_input_not_mutated_and_errors():
    A = gauss(60, 50, 1)
    before = A.copy()
    G.rqrcp(A, 20, b=8, p=4)
    G.trqrcp(A, 20, b=8, p=4)
    G.tuxv(A, 10, b=8, p=4)
    assert np.array_equal(A, before)
    with pytest.raises(ValueError):
        G.rqrcp(np.array([1.0, 2.0]), 1)
    with pytest.raises(ValueError):
        G.rqrcp(np.array([[np.nan, 1.0], [0.0, 1.0]]), 1)
    with pytest.raises(ValueError):
        G.rqrcp(np.eye(3), 4)
    with pytest.raises(ValueError):
        G.trqrcp(gauss(20, 16, 1), 12)
    with pytest.raises(ValueError):
        G.tuxv(gauss(20, 16, 1), 4, j_max=0)


def test_zero_and_rank_zero():
    assert G.rqrcp(np.zeros((10, 8), order="F"), 5, b=2, p=2).achieved_rank == 0
    assert G.trqrcp(np.zeros((12, 9), order="F"), 4, b=2, p=2).achieved_rank == 0
    res = G.tuxv(np.zeros((8, 6), order="F"), 3, b=2, p=1)
    assert res.achieved_rank == 0
    pf = G.rqrcp(np.eye(5), 0)
    assert pf.achieved_rank == 0 and pf.R.shape == (0, 5)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,b", [(2000, 1500, 1500, 64), (1200, 900, 300, 32), (700, 700, 650, 128)])
def test_rqrcp_streams_r_to_host(m, n, k, b):
    """rqrcp(..., out=R): R arrives on the host during the factorization and is
    identical to the device-materialised R; the strict lower part is untouched."""
    A = gauss(m, n, 21)
    ref = G.rqrcp(A, k, b=b, p=8, seed=0)
    out = np.zeros((min(k, m), n), order="F")
    got = G.rqrcp(A, k, b=b, p=8, seed=0, out=out)
    assert got.achieved_rank == ref.achieved_rank
    assert np.array_equal(got.perm, ref.perm)
    assert np.array_equal(got.R, ref.R)
    assert np.all(np.tril(out[: got.achieved_rank], -1) == 0.0)


@pytest.mark.parametrize("case", ["golden_rankdef", "p_block_exit", "j_block_exit", "noise_floor"])
def test_rqrcp_streams_r_to_host_rank_deficient(case):
    """out= on inputs whose last block is SHORT (bhat < bb): the trailing update
    of that block rewrites R rows of its own columns [i0+bhat, i0+bb), so the
    streamed R must leave only after the update (advisor finding, driver.cu RSink)."""
    if case == "golden_rankdef":
        g = load_golden("r_rankdef")
        A, kw = g["A"], golden_kwargs(g)
    else:
        r, seed, noise = {"p_block_exit": (39, 2, 0.0), "j_block_exit": (53, 1, 0.0),
                          "noise_floor": (61, 7, 1e-13)}[case]
        A = lowrank(200, 180, r, seed, noise)
        kw = dict(k=180, b=16, p=8, seed=seed)
    ref = G.rqrcp(A, **kw, omega="host")
    if case != "noise_floor":    # the noise-floor stop is rounding-ordered
        assert ref.achieved_rank < kw["k"]
    out = np.zeros((min(kw["k"], A.shape[0]), A.shape[1]), order="F")
    got = G.rqrcp(A, **kw, omega="host", out=out)
    assert got.achieved_rank == ref.achieved_rank
    assert np.array_equal(got.perm, ref.perm)
    assert np.array_equal(got.R, ref.R)
    if case != "noise_floor":   # at a 1e-13 noise floor the stopping pivot is rounding-ordered
        check_against(got, O.rqrcp(A, **kw), A, normwise=True)


def test_device_inputs_checked_and_untouched():
    """Column-major CUDA inputs go through the fused copy + finite scan
    (sqr_copy_check); tuxv reads A in place without modifying it; non-finite
    entries raise ValueError like validation.check_matrix."""
    A = gauss(300, 200, 4)
    Ad = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().T          # (m, n), stride (1, m)
    before = Ad.clone()
    pf = G.rqrcp(Ad, 100, b=16, p=8, omega="host")
    ref = O.rqrcp(A, 100, b=16, p=8, seed=0)
    assert np.array_equal(pf.perm, ref.perm)
    res = G.tuxv(Ad, 12, b=8, p=8, seed=1, omega="host")
    xref = O.tuxv(A, 12, b=8, p=8, seed=1)
    assert np.abs(res.reconstruct() - xref.reconstruct()).max() <= 1e-9 * np.abs(A).max()
    assert torch.equal(Ad, before)
    Cd = torch.from_numpy(A.copy()).cuda()                             # C-ordered: torch copy path
    assert np.array_equal(G.rqrcp(Cd, 100, b=16, p=8, omega="host").perm, ref.perm)
    for bad in (np.nan, np.inf, -np.inf):
        B = Ad.clone()
        B[7, 11] = bad
        with pytest.raises(ValueError, match="non-finite"):
            G.rqrcp(B, 10, b=8, p=4)
        with pytest.raises(ValueError, match="non-finite"):
            G.tuxv(B, 10, b=8, p=4)
        Bc = Cd.clone()
        Bc[3, 5] = bad
        with pytest.raises(ValueError, match="non-finite"):
            G.trqrcp(Bc, 10, b=8, p=4)


def lowrank(m, n, r, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    if noise:
        A += noise * rng.standard_normal((m, n))
    return np.asfortranarray(A)


# Early exits landing on the first (P, second sweep deferred) or the second
# (J, merged sweep) block of a pair: the paired second sweep must reproduce the
# reference's loop exits, R rows and counters exactly (driver.cu trailing_first /
# pending_panel_update / trailing_second).
@pytest.mark.parametrize("m,n,k,b,r,noise,seed", [
    (200, 180, 180, 16, 53, 0.0, 1),    # rank ends inside block 3 (a J block)
    (200, 180, 180, 16, 39, 0.0, 2),    # rank ends inside block 2 (a P block)
    (200, 180, 180, 16, 48, 0.0, 3),    # rank = 3 full blocks: sample floor at block 3
    (200, 180, 180, 16, 64, 0.0, 4),    # rank = 4 full blocks: exit after a complete pair
    (150, 170, 150, 16, 150, 0.0, 5),   # full rank, odd block count (10 blocks of 16, last 6 wide)
    (300, 130, 130, 12, 130, 0.0, 6),   # 11 blocks: the last one unpaired
    (120, 200, 100, 8, 60, 1e-13, 7),   # noise floor reached mid-pair
])
def test_paired_sweep_early_exits(m, n, k, b, r, noise, seed):
    A = lowrank(m, n, r, seed, noise)
    pf = G.rqrcp(A, k, b=b, p=8, seed=seed, omega="host")
    ref = O.rqrcp(A, k, b=b, p=8, seed=seed)
    check_against(pf, ref, A)
    if pf.achieved_rank:
        assert pf.rel_residual(A) <= 1e-12 * max(1.0, np.linalg.norm(A) / max(ref.r_diag[0], 1e-300))


def test_tuxv_wider_than_one_wy_kernel_block():
    """k > 144: the QLP factors are composed blocks wider than the fused
    apply kernel (factor._apply_blocks falls back to the chunked GEMMs)."""
    A = lowrank(420, 380, 170, 9, noise=1e-3)
    res = G.tuxv(A, 160, b=32, p=8, seed=4, omega="host", allow_large_k=True)
    ref = O.tuxv(A, 160, b=32, p=8, seed=4, allow_large_k=True)
    assert res.achieved_rank == ref.achieved_rank == 160
    assert np.abs(res.reconstruct() - ref.reconstruct()).max() <= 1e-9 * np.abs(A).max()
    U = res.u_columns()
    assert np.abs(U.T @ U - np.eye(160)).max() <= 1e-12


@pytest.mark.parametrize("same_stream", [False, True])
def test_concurrent_threads_disjoint_data(same_stream):
    """The reference's concurrency contract: calls from several threads on
    disjoint data are safe.  Two threads factor different
    matrices at once (own CUDA streams, or one shared stream); every result is
    bitwise equal to the same call made alone (deterministic kernels)."""
    import threading
    cases = [(gauss(900, 700, 50 + i), dict(k=600, b=32 + 32 * (i % 2), p=8, seed=i)) for i in range(4)]
    # alone first; the 4th case needs a larger workspace than the others (grow path)
    cases.append((gauss(3000, 2600, 60), dict(k=2600, b=128, p=8, seed=7)))
    alone = [G.rqrcp(A, **kw, omega="host") for A, kw in cases]
    want = [(pf.perm.copy(), pf.R.copy()) for pf in alone]
    tr = [G.trqrcp(A, 64, b=16, p=8, seed=3, omega="host") for A, _ in cases[:2]]
    want_t = [(tf.perm.copy(), tf.w_t.copy()) for tf in tr]
    errors = []
    shared = torch.cuda.Stream() if same_stream else None

    def worker(tid):
        try:
            s = shared if same_stream else torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    order = list(range(len(cases)))[tid::2] + list(range(len(cases)))[1 - tid::2]
                    for i in order:
                        A, kw = cases[i]
                        pf = G.rqrcp(A, **kw, omega="host")
                        if not (np.array_equal(pf.perm, want[i][0]) and np.array_equal(pf.R, want[i][1])):
                            errors.append(f"thread {tid} rep {rep} case {i}: rqrcp differs")
                    tf = G.trqrcp(cases[tid][0], 64, b=16, p=8, seed=3, omega="host")
                    if not (np.array_equal(tf.perm, want_t[tid][0]) and np.array_equal(tf.w_t, want_t[tid][1])):
                        errors.append(f"thread {tid} rep {rep}: trqrcp differs")
        except Exception as e:  # pragma: no cover - reported below
            errors.append(f"thread {tid}: {e!r}")

    ths = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors


@pytest.mark.parametrize("shape,kind", [((100, 100), "gauss"), ((300, 64), "gauss"), ((40, 90), "gauss"),
                                        ((80, 60), "rankdef"), ((33, 33), "decay"), ((20, 7), "zero")])
def test_jacobi_svd_matches_oracle(shape, kind):
    """Device one-sided Jacobi SVD (sqr_jacobi_svd) against the oracle's
    restatement of jacobi.py:50-117: singular values to 1e-12 relative, the
    same rotations (U, V equal to 1e-9), the rank-deficient completion
    orthonormal."""
    m, n = shape
    if kind == "gauss":
        A = gauss(m, n, 3)
    elif kind == "rankdef":
        A = np.asfortranarray(gauss(m, 17, 4) @ gauss(17, n, 5))
    elif kind == "decay":
        A = np.asfortranarray(O.synth_decay(m, n, 0.6, seed=2))
    else:
        A = np.zeros(shape, order="F")
    U, s, V = G.jacobi_svd(A)
    Ur, sr, Vr = O.jacobi_svd(A)
    k = min(m, n)
    assert U.shape == Ur.shape and V.shape == Vr.shape and s.shape == sr.shape
    if kind == "zero":
        assert np.array_equal(s, sr)
        return
    assert np.abs(s - sr).max() <= 1e-12 * sr[0]
    r = int(np.count_nonzero(sr > sr[0] * 1e-10))
    assert np.abs(U[:, :r] - Ur[:, :r]).max() <= 1e-9 and np.abs(V[:, :r] - Vr[:, :r]).max() <= 1e-9
    assert np.abs(U.T @ U - np.eye(k)).max() <= 1e-12
    assert np.abs((U * s) @ V.T - A).max() <= 1e-12 * sr[0]


def test_tuxv_refine_sigma_uses_jacobi():
    g = load_golden("x_refine")
    kw = golden_kwargs(g)
    kw["refine_sigma"] = True
    res = G.tuxv(g["A"], **kw, omega="host")
    assert np.abs(res.sigma_est - g["sigma_est"]).max() <= 1e-12 * g["sigma_est"].max()
    X = res.X
    assert np.abs(res.sigma_est - O.jacobi_svd(X)[1]).max() <= 1e-13 * res.sigma_est.max()


@pytest.mark.parametrize("fn,m,n,k,b,p,kind", [
    ("rqrcp", 700, 600, 600, 160, 8, "gauss"),      # b > 128: two sub-panels per block
    ("rqrcp", 900, 500, 400, 130, 20, "gauss"),     # b + p = 150 > 144
    ("rqrcp", 600, 520, 520, 300, 4, "lowrank"),    # rank 210 ends inside the second sub-panel
    ("rqrcp", 400, 380, 380, 256, 0, "zerocol"),    # exact zero columns: a short panel in sub-panel 2
    ("rsrqrcp", 800, 640, 640, 200, 8, "gauss"),
    ("trqrcp", 1000, 900, 420, 200, 8, "gauss"),
    ("trqrcp", 900, 800, 300, 140, 16, "decay"),
])
def test_wide_blocks_match_oracle(fn, m, n, k, b, p, kind):
    """Any b >= 1, p >= 0 (validation.py:75-82): blocks beyond the fused
    driver's 128 / 144 limits run the per-block loop of wide.py and must
    reproduce the reference loop (pivots, exits, R, w_t, counters)."""
    if kind == "gauss":
        A = gauss(m, n, 70)
    elif kind == "lowrank":
        A = lowrank(m, n, 210, 71)
    elif kind == "decay":
        A = np.asfortranarray(O.synth_decay(m, n, 10 ** (-8 / n), seed=3))
    else:
        A = gauss(m, n, 72)
        A[:, 150:] = 0.0
    extra = {} if fn == "rsrqrcp" else {"omega": "host"}
    got = getattr(G, fn)(A, k, b=b, p=p, seed=4, **extra)
    if fn == "rsrqrcp":   # device-drawn resamples: compare with the oracle fed the same draws is not possible;
        ref = O.rsrqrcp(A, k, b=b, p=p, seed=4)   # pivots agree away from ties (Gaussian input)
    else:
        ref = getattr(O, fn)(A, k, b=b, p=p, seed=4)
    check_against(got, ref, A, normwise=kind in ("lowrank", "zerocol", "decay"))
    if fn == "trqrcp":
        assert np.abs(got.w_t - ref.w_t).max() <= 1e-10 * np.abs(ref.w_t).max()
    if fn != "trqrcp" and got.achieved_rank == min(m, n):   # full factorizations: A P = Q R
        assert got.rel_residual(A) <= 1e-12
    elif got.achieved_rank:                                   # truncated: the reference's rank-r error
        assert abs(got.rel_residual(A, got.achieved_rank) - ref.rel_residual(A, got.achieved_rank)) <= \
            1e-10 * max(ref.rel_residual(A, got.achieved_rank), 1e-300) + 1e-13


@pytest.mark.parametrize("m,n,order", [(5000, 3001, "F"), (5001, 3000, "F"), (4000, 2500, "C"), (4001, 2499, "C")])
def test_pipelined_host_upload(m, n, order):
    """Large pageable host inputs go up through pinned staging chunks
    (_dev._h2d_pipelined), C-ordered ones transposed on the device: the device
    copy is bitwise the input, non-finite entries are still counted, and a
    factorization from the host array equals the one from a device tensor."""
    from paper_2008_04447_b200._dev import load_checked, upload
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n))
    A = np.asfortranarray(A) if order == "F" else np.ascontiguousarray(A)
    assert np.array_equal(upload(A, torch.device("cuda", 0)).numpy(), A)
    M = load_checked(A, torch.device("cuda", 0))
    assert np.array_equal(M.numpy(), A)
    B = A.copy(order=order)
    B[m // 2, n // 3] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        load_checked(B, torch.device("cuda", 0))
    if order == "C" and m == 4000:
        got = G.trqrcp(A, 40, b=16, p=8, seed=2, omega="host")
        dev = G.trqrcp(torch.from_numpy(A).cuda(), 40, b=16, p=8, seed=2, omega="host")
        assert np.array_equal(got.perm, dev.perm) and np.array_equal(got.w_t, dev.w_t)

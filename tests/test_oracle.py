"""Pin the CPU oracle (oracle/port.py) to the reference.

Two sources: the reference's own golden RNG values (pkg/tests/test_rng.py:31-67,
restated as literals here) and tests/golden/*.npz written by make_golden.py from
the real reference package.  Bit-exact where the reference is bit-exact
(RNG words, permutations, counters); outputs of BLAS-backed arithmetic are
compared bit-exactly too when produced on the same host, else to 1e-13.
"""
import numpy as np
import pytest

from conftest import gauss, golden_kwargs, load_golden
from oracle import port as O


def close(a, b, tol=1e-13):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    scale = max(1.0, float(np.abs(b).max()) if b.size else 1.0)
    assert float(np.abs(a - b).max() if a.size else 0.0) <= tol * scale


# --- RNG ------------------------------------------------------------------
def test_words_published_splitmix64():
    got = O.mix_words(0, np.arange(3, dtype=np.uint64))
    assert [hex(int(w)) for w in got] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4", "0x6c45d188009454f"]


def test_normals_reference_golden_values():
    assert O.gauss_stream(0, 6).tolist() == [
        -0.45275774021745807, 0.20776603893419174, 2.65060581207967,
        -0.49042282539864784, -0.9886041246243277, 1.8721013803315416]
    assert O.gauss_stream(12345, 4, offset=3).tolist() == [
        1.8429870753916229, -0.6061905461687912, 0.9957379931481631, -1.8615540099169032]


def test_rng_fixtures_bit_exact():
    g = load_golden("rng")
    assert np.array_equal(O.mix_words(0, np.arange(64, dtype=np.uint64)), g["words_seed0"])
    assert np.array_equal(O.mix_words(2**63 + 17, np.arange(64, dtype=np.uint64)), g["words_big"])
    assert np.array_equal(O.gauss_stream(0, 4096), g["normals_0_4096"])
    assert np.array_equal(O.gauss_stream(12345, 1000, offset=3), g["normals_12345_off3"])
    assert np.array_equal(O.gauss_matrix(40, 1000, 0), g["giid_40x1000_s0"])
    assert np.array_equal(O.gauss_matrix(72, 333, 7, offset=5), g["giid_72x333_s7_off5"])


def test_stream_cursor_and_offsets():
    s = O.GaussStream(11)
    head = s.draw_matrix(5, 2)
    tail = s.draw(5)
    whole = O.gauss_stream(11, 15)
    assert s.position == 15
    assert np.array_equal(head.flatten(order="F"), whole[:10]) and np.array_equal(tail, whole[10:])
    assert np.array_equal(O.gauss_stream(7, 100)[41:], O.gauss_stream(7, 59, offset=41))


# --- Householder ----------------------------------------------------------
def test_householder_kats():
    y, tau, beta = O.reflector(np.array([3.0, 4.0]))
    assert beta == -5.0 and np.allclose(y, [1.0, 0.5]) and np.isclose(tau, 1.6)
    y, tau, beta = O.reflector(np.array([1.0, 0.0]))
    assert (beta, tau) == (-1.0, 2.0)
    y, tau, beta = O.reflector(np.zeros(3))
    assert (tau, beta) == (0.0, 0.0) and y.tolist() == [1.0, 0.0, 0.0]
    g = load_golden("householder")
    for i in range(5):
        y, tau, beta = O.reflector(g[f"hg{i}_a"])
        close(y, g[f"hg{i}_y"], 0)
        close([tau, beta], g[f"hg{i}_tb"], 0)
    close(O.t_factor(g["wyT_Y"], g["wyT_tau"]), g["wyT_T"], 1e-15)


def test_downdate_kats():
    nsq, bad = O.downdate(np.array([25.0]), np.array([25.0]), np.array([3.0]))
    assert nsq.tolist() == [16.0] and not bad.any()
    r = 1.0 - 1e-13
    _, bad = O.downdate(np.array([1.0]), np.array([1.0]), np.array([r]))
    assert bad[0]


# --- deterministic QRCP ---------------------------------------------------
def _check_pf(pf, g, prefix="", tol=1e-13):
    assert np.array_equal(pf.perm, g[prefix + "perm"])
    assert pf.achieved_rank == int(g[prefix + "achieved"])
    assert [pf.counters.trailing_passes, pf.counters.blas2_volume, pf.counters.blas3_volume] == \
        g[prefix + "counters"].tolist()
    assert len(pf.blocks) == int(g[prefix + "nblocks"])
    close(pf.r_diag, g[prefix + "rdiag"], tol)
    if prefix + "R" in g:
        close(pf.R, g[prefix + "R"], tol)
    if prefix + "tau" in g:
        close(np.concatenate([b.tau for b in pf.blocks]), g[prefix + "tau"], tol)
        close(np.hstack([b.Y for b in pf.blocks]), g[prefix + "Ypack"], tol)
        close(pf.blocks[0].T, g[prefix + "T0"], tol)
    if prefix + "w_t" in g:
        close(pf.w_t, g[prefix + "w_t"], tol)


def test_qrcp_oracles_match_reference():
    g = load_golden("qrcp")
    A = g["qA"]
    _check_pf(O.qrcp_blas2(A), g, "blas2_")
    _check_pf(O.qrcp_blocked(A, b=8), g, "blocked_")
    _check_pf(O.qr_blocked(A, b=8), g, "qrb_")
    _check_pf(O.qrcp_blas2(np.diag([1.0, 2.0, 3.0])), g, "diag3_")
    _check_pf(O.qrcp_blas2(np.eye(4)), g, "eye4_")
    _check_pf(O.qrcp_blocked(np.diag(np.arange(1.0, 9.0)), b=4), g, "diag8_")
    assert O.qrcp_blas2(np.diag([1.0, 2.0, 3.0])).perm.tolist() == [2, 1, 0]


def test_sample_machinery_matches_reference():
    g = load_golden("sample")
    st = O.sample_pivots(g["sB"], 6)
    assert np.array_equal(st.local_perm, g["s_perm"]) and st.achieved == int(g["s_achieved"])
    close(st.B, g["s_B_out"])
    close(O.sample_refresh(st, g["s_R11"], g["s_R12"]), g["s_next"], 1e-12)
    assert np.array_equal(O.sample_pivots(g["tie_B"], 2).local_perm, g["tie_perm"])
    assert O.sample_pivots(g["tie_B"], 2).local_perm[0] == 0


DRIVER_CASES = ["r_small", "r_ragged", "r_tall", "r_wide", "r_short", "r_rankdef", "r_zero",
                "r_diag64", "r_kahan", "rs_small", "ss_small", "t_small", "t_decay", "t_short", "t_large_k"]


@pytest.mark.parametrize("name", DRIVER_CASES)
def test_drivers_match_reference(name):
    g = load_golden(name)
    kw = golden_kwargs(g)
    fn = {"r": O.rqrcp, "rs": O.rsrqrcp, "ss": O.ssrqrcp, "t": O.trqrcp}[name.split("_")[0]]
    if "allow_large_k" in kw:
        kw["allow_large_k"] = bool(kw["allow_large_k"])
    pf = fn(g["A"], **kw)
    _check_pf(pf, g, tol=1e-12)
    assert abs(pf.rel_residual(g["A"]) - float(g["rel_residual"])) <= 1e-13


@pytest.mark.parametrize("name", ["x_small", "x_flip2", "x_refine"])
def test_tuxv_matches_reference(name):
    g = load_golden(name)
    kw = golden_kwargs(g)
    if "refine_sigma" in kw:
        kw["refine_sigma"] = bool(kw["refine_sigma"])
    res = O.tuxv(g["A"], **kw)
    assert res.achieved_rank == int(g["achieved"])
    close(res.X, g["X"], 1e-12)
    close(res.sigma_est, g["sigma_est"], 1e-12)
    close(res.U.Y, g["UY"], 1e-12)
    close(res.V.Y, g["VY"], 1e-12)
    close(res.U.T, g["UT"], 1e-12)
    close(res.reconstruct(), g["recon"], 1e-12)
    assert [res.counters.trailing_passes, res.counters.blas2_volume, res.counters.blas3_volume] == \
        g["counters"].tolist()


@pytest.mark.slow
def test_config1_matches_reference():
    g = load_golden("c1")
    A = O.gauss_matrix(1000, 1000, 1)
    pf = O.rqrcp(A, 1000, b=32, p=8, seed=0)
    assert np.array_equal(pf.perm, g["perm"])
    close(pf.r_diag, g["rdiag"], 1e-12)
    assert [pf.counters.trailing_passes, pf.counters.blas2_volume, pf.counters.blas3_volume] == \
        g["counters"].tolist() == [62, 0, 705989120]


def test_omega_override_equals_stream():
    A = gauss(90, 70, 3)
    om = O.gauss_matrix(24, 90, 5)
    a = O.rqrcp(A, 40, b=16, p=8, seed=5)
    b = O.rqrcp(A, 40, b=16, p=8, seed=123, omega=om)
    assert np.array_equal(a.perm, b.perm) and np.array_equal(a.R, b.R)


def test_validation_errors():
    with pytest.raises(ValueError):
        O.rqrcp(np.array([1.0, 2.0]), 1)
    with pytest.raises(ValueError):
        O.rqrcp(np.array([[np.nan, 1.0], [0.0, 1.0]]), 1)
    with pytest.raises(ValueError):
        O.rqrcp(np.eye(3), 4)
    with pytest.raises(ValueError):
        O.rqrcp(np.eye(3), 2, b=0)
    with pytest.raises(ValueError):
        O.trqrcp(gauss(20, 16, 1), 12)
    with pytest.raises(ValueError):
        O.tuxv(gauss(20, 16, 1), 4, j_max=0)

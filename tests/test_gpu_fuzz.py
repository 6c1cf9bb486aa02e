"""Randomised parity sweep: RQRCP / RSRQRCP / TRQRCP / TUXV on the device against
the CPU oracle over seeded random shapes, block sizes, paddings, target ranks
and rank deficiencies (the north-star bars: identical pivots except at
documented near-ties, |R_jj| to 1e-10, residual <= 1e-12, identical counters,
truncated factors to 1e-10 / 1e-9)."""
import numpy as np
import pytest

from oracle import port as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2008_04447_b200 as G  # noqa: E402
from test_gpu_factor import check_against  # noqa: E402

NOISE = 1e-10


def check_fuzz(pf, ref, A):
    """check_against, except that for numerically rank-deficient inputs the
    STOP may fall at a different noise-floor pivot (the documented near-tie:
    the stopping tests compare rounding-level norms, and GPU sums are ordered
    differently): then everything above the noise floor must agree."""
    dr, d = np.abs(ref.r_diag), np.abs(pf.r_diag)
    floor = NOISE * dr[0] if dr.size else 0.0
    sig = int(np.count_nonzero(dr > floor))       # pivots above the noise floor (a prefix)
    if pf.achieved_rank == ref.achieved_rank and sig == ref.achieved_rank:
        check_against(pf, ref, A, noise=NOISE)  # no noise-floor pivots: the full bar
        return
    assert np.all(dr[sig:] <= floor) and np.all(d[sig:] <= floor), "achieved ranks differ above the noise floor"
    assert np.array_equal(pf.perm[:sig], ref.perm[:sig])
    assert np.all(np.abs(d[:sig] - dr[:sig]) <= 1e-10 * dr[:sig])


def draw(i):
    rng = np.random.default_rng(1000 + i)
    m = int(rng.integers(40, 700))
    n = int(rng.integers(30, 700))
    b = int(rng.choice([4, 8, 16, 24, 32, 64, 96, 128]))
    p = int(rng.choice([0, 2, 5, 8, 16]))
    kmax = min(m, n)
    k = int(rng.integers(1, kmax + 1))
    r = int(rng.integers(1, kmax + 1)) if rng.random() < 0.4 else kmax
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n)) if r < kmax else rng.standard_normal((m, n))
    if rng.random() < 0.3:  # graded column scaling
        A = A * (10.0 ** rng.uniform(-6, 0, size=n))
    return np.asfortranarray(A), k, b, p, int(rng.integers(0, 2**31))


@pytest.mark.parametrize("i", range(24))
def test_fuzz_rqrcp(i):
    A, k, b, p, seed = draw(i)
    if b + p > 144 or b > 128:
        pytest.skip("outside the kernel limits (b <= 128, b + p <= 144)")
    pf = G.rqrcp(A, k, b=b, p=p, seed=seed, omega="host")
    ref = O.rqrcp(A, k, b=b, p=p, seed=seed)
    check_fuzz(pf, ref, A)
    if pf.achieved_rank and pf.achieved_rank == ref.achieved_rank and np.array_equal(pf.perm, ref.perm):
        # same truncation error as the reference's factorization (1e-12 when it is complete)
        res, rres = pf.rel_residual(A), ref.rel_residual(A)
        assert abs(res - rres) <= 1e-12 + 1e-9 * rres


@pytest.mark.parametrize("i", range(24, 36))
def test_fuzz_trqrcp_tuxv(i):
    A, k, b, p, seed = draw(i)
    m, n = A.shape
    k = max(1, min(k, min(m, n) // 2))
    if b + p > 144 or b > 128:
        pytest.skip("outside the kernel limits")
    tf = G.trqrcp(A, k, b=b, p=p, seed=seed, omega="host")
    tref = O.trqrcp(A, k, b=b, p=p, seed=seed)
    if tf.achieved_rank != tref.achieved_rank:
        check_fuzz(tf, tref, A)  # stop at a different noise-floor pivot
        return
    j = np.nonzero(tf.perm != tref.perm)[0]
    if j.size == 0:
        scale = max(np.abs(tref.w_t).max(), 1e-300) if tref.w_t.size else 1.0
        assert np.abs(tf.w_t - tref.w_t).max() <= 1e-10 * scale
    res = G.tuxv(A, k, b=b, p=p, seed=seed, omega="host")
    xref = O.tuxv(A, k, b=b, p=p, seed=seed)
    assert res.achieved_rank == xref.achieved_rank
    if j.size == 0 and res.achieved_rank:
        assert np.abs(res.reconstruct() - xref.reconstruct()).max() <= 1e-9 * np.abs(A).max()


@pytest.mark.parametrize("i", range(36, 42))
def test_fuzz_rsrqrcp(i):
    A, k, b, p, seed = draw(i)
    if b + p > 144 or b > 128:
        pytest.skip("outside the kernel limits")
    pf = G.rsrqrcp(A, k, b=b, p=p, seed=seed)
    ref = O.rsrqrcp(A, k, b=b, p=p, seed=seed)
    check_fuzz(pf, ref, A)


EDGE = [
    # (m, n, k, b, p, rank)      what it reaches
    (50, 40, 40, 1, 0, 40),      # b = 1, p = 0
    (60, 50, 1, 16, 8, 50),      # k = 1
    (30, 60, 30, 32, 8, 30),     # l >= m: the blocked-QRCP fallback
    (200, 180, 180, 128, 16, 180),  # l = 144, the widest sample
    (150, 40000, 150, 16, 8, 150),  # n_t > 148*256: the shared-memory sample kernel
    (40000, 100, 100, 32, 8, 100),  # mr > 148*256: the leaf panel path
    (80000, 70, 70, 64, 8, 70),     # mr > 2*148*256: the generic panel kernel
    (300, 300, 300, 32, 8, 0),      # all-zero input
]


@pytest.mark.parametrize("case", EDGE, ids=lambda c: "x".join(map(str, c)))
def test_edge_shapes(case):
    m, n, k, b, p, r = case
    rng = np.random.default_rng(m * 7 + n)
    if r == 0:
        A = np.zeros((m, n), order="F")
    else:
        A = np.asfortranarray(rng.standard_normal((m, r)) @ rng.standard_normal((r, n)) if r < min(m, n)
                              else rng.standard_normal((m, n)))
    pf = G.rqrcp(A, k, b=b, p=p, seed=5, omega="host")
    ref = O.rqrcp(A, k, b=b, p=p, seed=5)
    check_fuzz(pf, ref, A)
    kt = max(1, min(k, min(m, n) // 2))
    tf = G.trqrcp(A, kt, b=b, p=p, seed=5, omega="host")
    tref = O.trqrcp(A, kt, b=b, p=p, seed=5)
    check_fuzz(tf, tref, A)


@pytest.mark.parametrize("j_max,refine", [(2, False), (3, True)])
def test_tuxv_flip_flops(j_max, refine):
    rng = np.random.default_rng(11)
    A = np.asfortranarray(rng.standard_normal((300, 40)) @ np.diag(0.7 ** np.arange(40)) @ rng.standard_normal((40, 260)))
    res = G.tuxv(A, 20, j_max=j_max, b=8, p=8, seed=2, refine_sigma=refine, omega="host")
    ref = O.tuxv(A, 20, j_max=j_max, b=8, p=8, seed=2, refine_sigma=refine)
    assert np.abs(res.reconstruct() - ref.reconstruct()).max() <= 1e-9 * np.abs(A).max()
    np.testing.assert_allclose(np.abs(res.sigma_est), np.abs(ref.sigma_est), rtol=1e-10)

"""The reference's callers bound to the B200 path (paper_2008_04447_b200/callers.py):
experiment dispatch / counters / quality records and the scikit-learn wrappers,
against golden outputs of the real reference (tests/golden/make_golden_callers.py)
and the behaviours its own tests pin (test_estimators.py, test_quality_cli.py)."""
import numpy as np
import pytest

from conftest import load_golden

from paper_2008_04447_b200 import callers as C


def test_lower_median_and_rank_grid():
    assert C.lower_median([3.0, 1.0, 2.0, 4.0]) == 2.0
    assert C.lower_median([5.0]) == 5.0
    with pytest.raises(ValueError):
        C.lower_median([])
    assert C.rank_grid(64, 32) == [32, 64]
    assert C.rank_grid(65, 32) == [32, 64]
    assert C.rank_grid(20, 32) == [20]
    assert set(C.DETERMINISTIC_ALGORITHMS) <= set(C.ALGORITHMS)


torch = pytest.importorskip("torch")
gpu = pytest.mark.gpu
needs_cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs CUDA")


@gpu
@needs_cuda
def test_presort_orders_by_norm():
    A = np.array([[1.0, 3.0, 2.0]], order="F")
    s, order = C.presort_columns(A)
    np.testing.assert_array_equal(order, [1, 2, 0])
    np.testing.assert_array_equal(s, [[3.0, 2.0, 1.0]])


@gpu
@needs_cuda
@pytest.mark.parametrize("algo", ["qrcp", "qrcp_blocked", "ssrqrcp", "rqrcp", "rsrqrcp", "trqrcp"])
def test_randomized_pivoted_qr_matches_reference(algo):
    g = load_golden("callers")
    X = g["X"]
    est = C.RandomizedPivotedQR(rank=9, algorithm=algo, block_size=4, padding=4, random_state=5,
                                omega="host").fit(X)
    np.testing.assert_array_equal(est.selected_columns_, g[f"est_{algo}_sel"])
    np.testing.assert_array_equal(est.permutation_, g[f"est_{algo}_perm"])
    np.testing.assert_allclose(est.r_diagonal_, g[f"est_{algo}_rdiag"], rtol=1e-10, atol=1e-12)
    assert est.rank_ == 9 and est.n_features_in_ == 40
    np.testing.assert_array_equal(est.transform(X), X[:, est.selected_columns_])


@gpu
@needs_cuda
def test_truncated_qlp_matches_reference():
    g = load_golden("callers")
    X = g["X"]
    q = C.TruncatedQLP(rank=6, block_size=4, padding=4, random_state=3, omega="host")
    Xt = q.fit_transform(X)
    np.testing.assert_allclose(q.singular_values_, g["qlp_sv"], rtol=1e-10)
    np.testing.assert_allclose(q.middle_, g["qlp_middle"], atol=1e-10)
    np.testing.assert_allclose(q.components_, g["qlp_components"], atol=1e-9)
    np.testing.assert_allclose(Xt, g["qlp_Xt"], atol=1e-9)
    np.testing.assert_allclose(q.inverse_transform(q.transform(X)), (X @ q.components_.T) @ q.components_,
                               atol=1e-12)
    q2 = C.TruncatedQLP(rank=6, flip_flops=2, block_size=4, padding=4, refine_sigma=False, random_state=3,
                        omega="host").fit(X)
    np.testing.assert_allclose(q2.singular_values_, g["qlp2_sv"], rtol=1e-10)


@gpu
@needs_cuda
def test_run_counters_match_reference():
    g = load_golden("callers")
    A = g["A"]
    for algo, want in zip(g["counters_algos"], g["counters"]):
        c = C.run_counters(A, str(algo), rank=16, block=8, pad=4, seed=7, omega="host")
        got = [c["achieved_rank"], c["trailing_passes"], c["blas2_volume"], c["blas3_volume"]]
        assert got == want.tolist(), algo
    with pytest.raises(ValueError):
        C.run_counters(np.eye(8), "svd", rank=4)


@gpu
@needs_cuda
def test_run_quality_matches_reference():
    g = load_golden("callers")
    A = g["A"]
    for algo, want in zip(g["quality_algos"], g["quality"]):
        recs = C.run_quality(A, str(algo), rank=24, block=8, pad=4, seed=3, reps=3, omega="host")
        got = np.array([[r.rank, r.reps, r.err_min, r.err_median, r.err_max] for r in recs])
        np.testing.assert_array_equal(got[:, :2], want[:, :2])
        np.testing.assert_allclose(got[:, 2:], want[:, 2:], rtol=1e-8, atol=1e-13, err_msg=str(algo))
    with pytest.raises(ValueError):
        C.run_quality(A, "cholesky", rank=8)
    with pytest.raises(ValueError):
        C.run_quality(np.zeros((8, 8)), "rqrcp", rank=4)


@gpu
@needs_cuda
def test_estimator_behaviour():
    from sklearn.base import clone
    from sklearn.exceptions import NotFittedError
    from sklearn.pipeline import make_pipeline
    X = load_golden("callers")["X"]
    with pytest.raises(NotFittedError):
        C.RandomizedPivotedQR(rank=3).transform(X)
    for bad in (dict(rank=0), dict(rank=41), dict(rank=3, algorithm="cholesky")):
        with pytest.raises(ValueError):
            C.RandomizedPivotedQR(**bad).fit(X)
    est = C.RandomizedPivotedQR(rank=4, random_state=0).fit(X)
    with pytest.raises(ValueError):
        est.transform(X[:, :20])
    a = C.RandomizedPivotedQR(rank=8, algorithm="qrcp", random_state=1).fit(X)
    b = C.RandomizedPivotedQR(rank=8, algorithm="qrcp", random_state=2).fit(X)
    np.testing.assert_array_equal(a.selected_columns_, b.selected_columns_)
    e = C.RandomizedPivotedQR(rank=9, algorithm="trqrcp", block_size=4, padding=2, random_state=5)
    dup = clone(e)
    assert dup.get_params() == e.get_params()
    np.testing.assert_array_equal(dup.fit(X).selected_columns_, e.fit(X).selected_columns_)
    pipe = make_pipeline(C.RandomizedPivotedQR(rank=5, random_state=0), C.TruncatedQLP(rank=3, random_state=0))
    assert pipe.fit_transform(X).shape == (60, 3)

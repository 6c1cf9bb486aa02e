"""The reference's callers of the hot path, bound to the B200 factorizations
(SURVEY.md §8(f) rank 4): the experiment-layer dispatch and metrics of
``sketchqr.quality`` (quality.py:44-178) and the scikit-learn wrappers of
``sketchqr.estimators`` (estimators.py:23-186).  Same names, arguments,
defaults, result records and error types; every factorization, residual and
reconstruction runs on the device.  CSV/CLI plumbing stays out of scope.

``omega`` (extra, default None = the device stream) is forwarded to the
factorizations that accept it; ``omega="host"`` reproduces the reference's
host Omega bit for bit (the parity tests use it).
"""
from __future__ import annotations

import numbers
from dataclasses import dataclass

import numpy as np
import torch

from . import factor as F
from ._dev import require_cuda, upload

__all__ = [
    "ALGORITHMS", "DETERMINISTIC_ALGORITHMS", "QualityRecord", "lower_median", "rank_grid", "presort_columns",
    "make_factorization", "run_quality", "run_counters", "RandomizedPivotedQR", "TruncatedQLP",
]

# quality.py:42-43
ALGORITHMS = ("qrcp2", "qrcp3", "qr", "ssrqrcp", "rqrcp", "rsrqrcp", "trqrcp", "tuxv", "svd")
DETERMINISTIC_ALGORITHMS = frozenset({"qrcp2", "qrcp3", "qr", "svd"})


@dataclass
class QualityRecord:
    """quality.py:68-75."""

    algorithm: str
    rank: int
    reps: int
    err_min: float
    err_median: float
    err_max: float


def lower_median(values) -> float:
    """quality.py:78-82: the lower median (even counts take the smaller)."""
    s = sorted(values)
    if not s:
        raise ValueError("median of empty sequence")
    return s[(len(s) - 1) // 2]


def rank_grid(k: int, b: int) -> list[int]:
    """quality.py:85-87: {b, 2b, ...} <= k, or [k] when k < b."""
    grid = list(range(b, k + 1, b))
    return grid or [k]


def presort_columns(A):
    """quality.py:90-93: columns in descending 2-norm order (stable) and the
    order applied.  Norms on the device; returns a host Fortran array like the
    reference when given one, else a device (m, n) column-major view."""
    dev = require_cuda(A.device if isinstance(A, torch.Tensor) and A.is_cuda else None)
    M = upload(A, dev)
    norms = torch.linalg.vector_norm(M.view(), dim=0)
    order = torch.sort(-norms, stable=True).indices
    Ms = M.view()[:, order]
    order_h = order.cpu().numpy().astype(np.int64)
    if isinstance(A, torch.Tensor):
        return Ms, order_h
    return np.asfortranarray(Ms.cpu().numpy()), order_h


def _presorted_qr(A, k, b):
    As, order = presort_columns(A)
    pf = F.qr_blocked(As, k, b)
    pf.perm = order
    return pf


# quality.py names -> device call (A, k, b, p, seed, omega, presort)
_FACTORIZATIONS = {
    "qrcp2": lambda A, k, b, p, s, om, ps: F.qrcp_blas2(A, k),
    "qrcp3": lambda A, k, b, p, s, om, ps: F.qrcp_blocked(A, k, b),
    "qr": lambda A, k, b, p, s, om, ps: _presorted_qr(A, k, b) if ps else F.qr_blocked(A, k, b),
    "ssrqrcp": lambda A, k, b, p, s, om, ps: F.ssrqrcp(A, k, p=p, seed=s, omega=om),
    "rqrcp": lambda A, k, b, p, s, om, ps: F.rqrcp(A, k, b=b, p=p, seed=s, omega=om),
    "rsrqrcp": lambda A, k, b, p, s, om, ps: F.rsrqrcp(A, k, b=b, p=p, seed=s),
    "trqrcp": lambda A, k, b, p, s, om, ps: F.trqrcp(A, k, b=b, p=p, seed=s, allow_large_k=True, omega=om),
}


def make_factorization(A, algorithm, k, b, p, seed, presort_qr: bool = False, omega=None):
    """quality.py:96-117 (qrcp2 = BLAS-2 QRCP, qrcp3 = blocked QRCP, qr =
    unpivoted blocked QR, optionally on norm-presorted columns)."""
    make = _FACTORIZATIONS.get(algorithm)
    if make is None:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    return make(A, k, b, p, seed, omega, presort_qr)


def _device_matrix(A):
    dev = require_cuda(A.device if isinstance(A, torch.Tensor) and A.is_cuda else None)
    return upload(A, dev).view()


def run_quality(A, algorithm: str, rank: int, block: int = 32, pad: int = 8, seed: int = 0, reps: int = 100,
                omega=None) -> list[QualityRecord]:
    """quality.py:120-162: relative Frobenius errors over the rank grid, min /
    lower-median / max over `reps` seeded repetitions (one for the
    deterministic algorithms).  "svd" rows are the Eckart-Young errors from the
    singular values of the device Jacobi SVD (sqr_jacobi_svd; the reference
    forms U diag(s) V^T of its Jacobi SVD, the same optimal rank-r errors to
    rounding)."""
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    Ad = _device_matrix(A)
    fro = float(torch.linalg.norm(Ad))
    if fro == 0.0:
        raise ValueError("quality of an all-zero matrix is not meaningful")
    ranks = rank_grid(rank, block)
    reps_eff = 1 if algorithm in DETERMINISTIC_ALGORITHMS else max(1, reps)
    errs: dict[int, list[float]] = {r: [] for r in ranks}
    if algorithm == "svd":
        if min(Ad.shape) <= 4096:   # the reference's Jacobi SVD (quality.py:133), on the device
            W = F.ColMajor.empty(*Ad.shape, Ad.device) if Ad.shape[0] >= Ad.shape[1] else None
            if W is not None:
                W.view().copy_(Ad)
            else:
                W = F.ColMajor.empty(Ad.shape[1], Ad.shape[0], Ad.device)
                W.view().copy_(Ad.T)
            s = F._jacobi_svd_dev(W)[1]
        else:
            s = torch.linalg.svdvals(Ad)
        tail = torch.flip(torch.cumsum(torch.flip(s * s, [0]), 0), [0])  # tail[r] = sum_{i >= r} s_i^2
        for r in ranks:
            errs[r].append(float(torch.sqrt(tail[r]) / fro) if r < s.numel() else 0.0)
    elif algorithm == "tuxv":
        for rep in range(reps_eff):
            for r in ranks:
                res = F.tuxv(Ad, r, b=block, p=pad, seed=seed + rep, allow_large_k=True, omega=omega)
                errs[r].append(float(torch.linalg.norm(Ad - res.reconstruct_device()) / fro))
    else:
        for rep in range(reps_eff):
            pf = make_factorization(Ad, algorithm, rank, block, pad, seed + rep, presort_qr=True, omega=omega)
            for r in ranks:
                errs[r].append(float(torch.linalg.norm(Ad - pf._reconstruct_dev(r)) / fro))
    return [QualityRecord(algorithm, r, reps_eff, min(errs[r]), lower_median(errs[r]), max(errs[r]))
            for r in ranks]


def run_counters(A, algorithm: str, rank: int, block: int = 32, pad: int = 8, seed: int = 0, omega=None) -> dict:
    """quality.py:165-178: communication counters of one run."""
    if algorithm == "svd":
        raise ValueError("counters are tracked for the QR-family algorithms only")
    if algorithm == "tuxv":
        result = F.tuxv(A, rank, b=block, p=pad, seed=seed, allow_large_k=True, omega=omega)
        counters, achieved = result.counters, result.achieved_rank
    else:
        pf = make_factorization(A, algorithm, rank, block, pad, seed, omega=omega)
        counters, achieved = pf.counters, pf.achieved_rank
    m, n = A.shape
    return {"algorithm": algorithm, "m": m, "n": n, "rank": rank, "achieved_rank": achieved, "block": block,
            "pad": pad, "seed": seed, "trailing_passes": counters.trailing_passes,
            "blas2_volume": counters.blas2_volume, "blas3_volume": counters.blas3_volume}


# ---------------------------------------------------------------- sklearn
try:  # the wrappers need scikit-learn, like the reference's estimators module
    from sklearn.base import BaseEstimator, TransformerMixin
    from sklearn.utils import check_array, check_random_state
    from sklearn.utils.validation import check_is_fitted
except ImportError:  # pragma: no cover
    BaseEstimator = TransformerMixin = object
    check_array = check_random_state = check_is_fitted = None


def _seed_of(random_state) -> int:
    """estimators.py:33-40: an integer feeds the counter-based stream as is
    (masked to 64 bits); anything else draws one through sklearn."""
    if isinstance(random_state, numbers.Integral):
        return int(random_state) & 0xFFFFFFFFFFFFFFFF
    return int(check_random_state(random_state).randint(0, 2**63 - 1))


# estimators.py:23-30 names -> device call (X, k, b, p, seed, omega); the QRCP
# oracles ignore the seed, trqrcp is called with allow_large_k like the reference
_SELECTORS = {
    "qrcp": lambda X, k, b, p, s, om: F.qrcp_blas2(X, k),
    "qrcp_blocked": lambda X, k, b, p, s, om: F.qrcp_blocked(X, k, b),
    "ssrqrcp": lambda X, k, b, p, s, om: F.ssrqrcp(X, k, p=p, seed=s, omega=om),
    "rqrcp": lambda X, k, b, p, s, om: F.rqrcp(X, k, b=b, p=p, seed=s, omega=om),
    "rsrqrcp": lambda X, k, b, p, s, om: F.rsrqrcp(X, k, b=b, p=p, seed=s),
    "trqrcp": lambda X, k, b, p, s, om: F.trqrcp(X, k, b=b, p=p, seed=s, allow_large_k=True, omega=om),
}


class _DeviceTransformer(TransformerMixin, BaseEstimator):
    """Shared input handling of the two wrappers."""

    def _fit_input(self, X):
        X = check_array(X, dtype=np.float64, order="F")
        k = int(self.rank)
        if k < 1 or k > min(X.shape):
            raise ValueError(f"rank must be in [1, min(m, n)], got {k}")
        return X, k

    def _new_input(self, X, attr):
        check_is_fitted(self, attr)
        X = check_array(X, dtype=np.float64)
        if X.shape[1] != self.n_features_in_:
            raise ValueError(f"X has {X.shape[1]} features, expected {self.n_features_in_}")
        return X


class RandomizedPivotedQR(_DeviceTransformer):
    """Column subset selection by a pivoted factorization on the device
    (estimators.py:43-126): `transform` keeps the rank_ leading pivot columns."""

    def __init__(self, rank=8, algorithm="rqrcp", block_size=32, padding=8, random_state=None, omega=None):
        self.rank = rank
        self.algorithm = algorithm
        self.block_size = block_size
        self.padding = padding
        self.random_state = random_state
        self.omega = omega

    def fit(self, X, y=None):
        X = check_array(X, dtype=np.float64, order="F")
        select = _SELECTORS.get(self.algorithm)
        if select is None:
            raise ValueError(f"algorithm must be one of {sorted(_SELECTORS)}, got {self.algorithm!r}")
        X, k = self._fit_input(X)
        pf = select(X, k, int(self.block_size), int(self.padding), _seed_of(self.random_state), self.omega)
        self.factorization_ = pf
        self.rank_ = pf.achieved_rank
        self.permutation_ = np.array(pf.perm, copy=True)
        self.selected_columns_ = self.permutation_[: self.rank_].copy()
        self.r_diagonal_ = np.array(pf.r_diag, copy=True)
        self.n_features_in_ = X.shape[1]
        return self

    def transform(self, X):
        return self._new_input(X, "selected_columns_")[:, self.selected_columns_]


def _device_matmul(A, B) -> np.ndarray:
    """A @ B on the device (libsqr DMMA GEMM), NumPy out: the estimator's
    projections (estimators.py:157-186) stay off the host like every other
    product of this package."""
    dev = require_cuda()
    return F.gemm_nn(upload(A, dev), upload(B, dev)).numpy()


class TruncatedQLP(_DeviceTransformer):
    """TruncatedSVD-like surface over TUXV (estimators.py:129-186):
    components_ = V^T, singular_values_ = sigma_est, middle_ = X."""

    def __init__(self, rank=8, flip_flops=1, block_size=32, padding=8, refine_sigma=True, random_state=None,
                 omega=None):
        self.rank = rank
        self.flip_flops = flip_flops
        self.block_size = block_size
        self.padding = padding
        self.refine_sigma = refine_sigma
        self.random_state = random_state
        self.omega = omega

    def fit(self, X, y=None):
        self.fit_transform(X, y)
        return self

    def fit_transform(self, X, y=None):
        X, k = self._fit_input(X)
        res = F.tuxv(X, k, j_max=int(self.flip_flops), b=int(self.block_size), p=int(self.padding),
                     seed=_seed_of(self.random_state), refine_sigma=bool(self.refine_sigma), allow_large_k=True,
                     omega=self.omega)
        V = res.v_columns()
        self.result_, self.rank_ = res, res.achieved_rank
        self.components_ = np.ascontiguousarray(V.T)
        self.singular_values_ = np.array(res.sigma_est, copy=True)
        self.middle_ = np.array(res.X, copy=True)
        self.n_features_in_ = X.shape[1]
        return _device_matmul(X, V)

    def transform(self, X):
        return _device_matmul(self._new_input(X, "components_"), self.components_.T)

    def inverse_transform(self, X):
        check_is_fitted(self, "components_")
        return _device_matmul(check_array(X, dtype=np.float64), self.components_)

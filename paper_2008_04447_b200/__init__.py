"""B200-native randomized column-pivoted QR (Duersch & Gu, arXiv 2008.04447).

Drop-in for the hot path of the reference package ``sketchqr``: the same
rqrcp / rsrqrcp / ssrqrcp / trqrcp / tuxv call signatures and result types
(plus the deterministic qrcp_blocked / qrcp_blas2 / qr_blocked they fall
back on), executed by hand-written sm_100a kernels in ``libsqr.so``.
"""
__version__ = "0.1.0"

from .counters import CommCounters
from .factor import (PivotedFactorization, ReflectorBlock, TruncatedFactorization, TuxvResult, apply_blocks_q,
                     apply_blocks_qt, blocks_q_columns, invert_permutation, jacobi_svd, qr_blocked, qrcp_blas2, qrcp_blocked,
                     rqrcp, rsrqrcp, ssrqrcp, trqrcp, tuxv, wy_compose)
from .rng import NormalStream, device_giid, giid, normals
from . import callers  # noqa: E402  (quality / estimators callers of the hot path)

__all__ = [
    "CommCounters", "PivotedFactorization", "ReflectorBlock", "TruncatedFactorization", "TuxvResult",
    "apply_blocks_q", "apply_blocks_qt", "blocks_q_columns", "invert_permutation", "jacobi_svd", "qr_blocked", "qrcp_blas2",
    "qrcp_blocked", "rqrcp", "rsrqrcp", "ssrqrcp", "trqrcp", "tuxv", "wy_compose", "NormalStream",
    "device_giid", "giid", "normals",
]

"""CPU checks of the drop-in boundary: libsqr.so loads and exports every
symbol include/sqr.h declares; the ctypes table matches the header."""
import os
import re

import pytest

from paper_2008_04447_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sqr.h")).read()
    return sorted(set(re.findall(r"\b(sqr_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_binding_table():
    assert header_symbols() == sorted(_lib.exported_symbols())


def test_library_exports_every_symbol():
    L = _lib.lib()
    for name in header_symbols():
        assert hasattr(L, name), name
    assert b"sm_100a" in L.sqr_version()


def test_workspace_queries_without_gpu():
    L = _lib.lib()
    w = L.sqr_rqrcp_workspace(32768, 32768, 32768, 128, 8)
    assert 0 < w < 2 << 30
    assert L.sqr_trqrcp_workspace(20000, 20000, 100, 32, 8) > 0
    assert L.sqr_qr_blocked_workspace(20000, 100, 100, 32) > 0


def test_status_layout():
    assert _lib.STATUS_BYTES == 72  # static_assert in driver.cu


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2008_04447_b200 as G
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        G.rqrcp(np.eye(40), 4, b=2, p=2)

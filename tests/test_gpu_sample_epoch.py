"""Pivot-epoch sample QRCP (csrc/sample_epoch.cu) against the thread-per-column
kernel it replaces and against the oracle (reference.py:107-150 via
sketch.py:97-119).

The epoch kernel runs the pivot steps on a leader CTA over the best <= 224
candidate columns and only while the winner provably beats every other column;
its per-column arithmetic repeats the per-pivot-barrier kernel's (the reflector
norm is summed in a different order).  So on every input -- including
adversarial ones for the candidate bound (graded columns concentrated in one
worker, exact ties, duplicated and zero columns, low rank) -- it must give the
same stop status and |R| diagonal as that kernel (SQR_EPOCH_SAMPLE=1 selects
the epoch kernel; the switch is read per call), the same pivots wherever the columns are not
tied to rounding, and on well-separated inputs the oracle's pivots.
"""
import os

import numpy as np
import pytest

from conftest import gauss
from oracle import port as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2008_04447_b200 import _lib  # noqa: E402
from paper_2008_04447_b200._dev import ColMajor, status_new, status_read, stream_handle, upload  # noqa: E402

DEV = torch.device("cuda", 0)
L = _lib.lib()


def run_sample(B, bb, first=1, epoch=True, floor_sq=None):
    ell, nt = B.shape
    old = os.environ.get("SQR_EPOCH_SAMPLE")
    if epoch:
        os.environ["SQR_EPOCH_SAMPLE"] = "1"
    else:
        os.environ.pop("SQR_EPOCH_SAMPLE", None)
    try:
        Bd = upload(np.asfortranarray(B), DEV)
        Bf = ColMajor.empty(ell, nt, DEV)
        lperm = torch.full((nt,), -7, dtype=torch.int64, device=DEV)
        moves = torch.full((4 * bb + 8,), -9, dtype=torch.int32, device=DEV)
        taus = torch.zeros(max(bb, 1), dtype=torch.float64, device=DEV)
        st = status_new(DEV)
        if floor_sq is not None:
            off = _lib.STATUS_DTYPE.fields["floor_sq"][1]
            st[off:off + 8].copy_(torch.tensor([floor_sq], dtype=torch.float64).view(torch.uint8).to(DEV))
        _lib.check(L.sqr_sample_qrcp(Bd.ptr, Bd.ld, ell, nt, bb, Bf.ptr, Bf.ld, lperm.data_ptr(), moves.data_ptr(),
                                     taus.data_ptr(), first, st.data_ptr(), stream_handle()))
        torch.cuda.synchronize()
        s = status_read(st)
        nm = int(s["nmoves"])
        return {"Bf": Bf.numpy(), "lperm": lperm.cpu().numpy(), "taus": taus.cpu().numpy(),
                "moves": moves.cpu().numpy()[: 2 * nm],
                "status": {k: np.asarray(s[k]).tolist() for k in _lib.STATUS_DTYPE.names}}
    finally:
        if old is None:
            os.environ.pop("SQR_EPOCH_SAMPLE", None)
        else:
            os.environ["SQR_EPOCH_SAMPLE"] = old


def assert_same(a, b, exact_pivots=True):
    assert a["status"] == b["status"]
    if a["status"]["stop"] and a["status"]["reason"] == 2:
        return  # sample-floor stop before the first pivot: no outputs are defined
    k = int(a["status"]["sample_achieved"])
    da, db = np.abs(np.diag(a["Bf"][:k, :k])), np.abs(np.diag(b["Bf"][:k, :k]))
    scale = max(db.max() if k else 0.0, 1e-300)
    assert np.abs(da - db).max(initial=0.0) <= 1e-10 * scale
    if not exact_pivots:
        # ties to rounding: any tied column may win; the permutation is valid
        assert np.array_equal(np.sort(a["lperm"]), np.arange(a["lperm"].size))
        return
    assert np.array_equal(a["lperm"], b["lperm"])
    assert np.array_equal(a["moves"], b["moves"])
    assert np.abs(a["taus"] - b["taus"]).max(initial=0.0) <= 1e-12
    assert np.abs(a["Bf"] - b["Bf"]).max() <= 1e-11 * max(np.abs(b["Bf"]).max(), 1e-300)


def _graded(ell, nt, seed, rate):
    B = gauss(ell, nt, seed)
    return np.asfortranarray(B * np.exp(-rate * np.arange(nt) / nt)[None, :])


def _cases():
    rng = np.random.default_rng(11)
    c = {}
    c["g1_small"] = (gauss(40, 100, 1), 32)
    c["g1_full"] = (gauss(136, 256, 2), 128)
    c["g2"] = (gauss(136, 257, 3), 128)
    c["g4"] = (gauss(72, 1000, 4), 64)
    c["g20"] = (gauss(136, 5000, 5), 128)
    c["g128"] = (gauss(136, 32768, 6), 128)
    c["g147"] = (gauss(136, 147 * 256, 7), 128)
    c["ell144"] = (gauss(144, 9000, 8), 128)
    c["ell9"] = (gauss(9, 3000, 9), 9)
    c["ell47"] = (gauss(47, 2000, 10), 40)
    # candidate bound stress: every large column in one worker (first / last)
    c["graded_first"] = (_graded(136, 8000, 12, 30.0), 128)
    c["graded_last"] = (np.asfortranarray(_graded(136, 8000, 13, 30.0)[:, ::-1]), 128)
    c["graded_mild"] = (_graded(72, 20000, 14, 0.5), 64)
    # exact ties: duplicated columns, +-1 entries (all initial norms equal)
    base = gauss(72, 50, 15)
    c["dup"] = (np.asfortranarray(base[:, np.arange(6000) % 50]), 64)
    c["pm1"] = (np.asfortranarray(np.where(rng.random((40, 3000)) < 0.5, -1.0, 1.0)), 32)
    # low rank, zero columns
    c["rank10"] = (np.asfortranarray(gauss(72, 10, 16) @ gauss(10, 4000, 17)), 64)
    Z = np.zeros((40, 5000), order="F")
    Z[:, ::997] = gauss(40, Z[:, ::997].shape[1], 18)
    c["sparse_cols"] = (Z, 32)
    c["zero"] = (np.zeros((40, 1000), order="F"), 32)
    return c


CASES = _cases()


TIED = {"pm1", "rank10", "sparse_cols", "zero"}


@pytest.mark.parametrize("name", sorted(CASES))
def test_epoch_equals_per_pivot_kernel(name):
    B, bb = CASES[name]
    bb = min(bb, B.shape[0], B.shape[1])
    got = run_sample(B, bb, epoch=True)
    want = run_sample(B, bb, epoch=False)
    assert_same(got, want, exact_pivots=name not in TIED)


@pytest.mark.parametrize("name", ["g1_small", "g1_full", "g2", "g4", "g20", "g128", "g147", "ell144", "ell9",
                                  "graded_first", "graded_last", "graded_mild"])
def test_epoch_matches_oracle(name):
    B, bb = CASES[name]
    bb = min(bb, B.shape[0], B.shape[1])
    got = run_sample(B, bb)
    ref = O.sample_pivots(B, bb)
    assert int(got["status"]["sample_achieved"]) == ref.achieved
    assert np.array_equal(got["lperm"], ref.local_perm)
    a = ref.achieved
    Bf = got["Bf"]
    scale = np.abs(ref.S11).max()
    assert np.abs(np.triu(Bf[:a, :a]) - ref.S11).max() <= 1e-12 * scale
    assert np.abs(got["taus"][:a] - ref.u_block.tau).max() <= 1e-12


def test_epoch_not_first_uses_status_floor():
    """first=0: the sample floor comes from the status word (randomized.py:188-190)."""
    B = gauss(40, 3000, 21)
    mx = float((B * B).sum(0).max())
    got = run_sample(B, 32, first=0, floor_sq=2.0 * mx)   # everything below the floor: stop
    assert got["status"]["stop"] == 1 and got["status"]["reason"] == 2
    got = run_sample(B, 32, first=0, floor_sq=1e-300)
    want = run_sample(B, 32, first=0, floor_sq=1e-300, epoch=False)
    assert_same(got, want)
    assert got["status"]["sample_achieved"] == 32


@pytest.mark.parametrize("name", ["g128", "pm1", "dup"])
def test_epoch_repeatable(name):
    """Bitwise run-to-run determinism (fixed-order reductions everywhere)."""
    B, bb = CASES[name]
    bb = min(bb, B.shape[0], B.shape[1])
    a = run_sample(B, bb)
    b = run_sample(B, bb)
    assert a["status"] == b["status"]
    for k in ("lperm", "taus", "moves", "Bf"):
        assert np.array_equal(a[k], b[k])

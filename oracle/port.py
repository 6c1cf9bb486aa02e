"""CPU oracle: a NumPy restatement of the reference ``sketchqr`` hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2008_04447_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs do, and there only as the checker
or as the timed CPU baseline.  The product path is the CUDA library.

Every routine below restates the reference algorithm (cited as
``pkg/src/sketchqr/<file>:<line>``) with the same NumPy call shapes and the same
order of floating-point operations, so on one host its outputs are bit-identical
to the reference's.  That claim is pinned by ``tests/golden/*.npz`` (written by
``tests/golden/make_golden.py`` from the real reference in the build container)
and by the reference's own golden RNG values (``pkg/tests/test_rng.py:31-67``),
both checked in ``tests/test_oracle.py``.

Two extension points the reference does not have, used by the GPU parity tests:

* ``omega=``: feed an explicit sketch matrix (l x m) instead of drawing it
  from the seed's stream, so the oracle can be run on exactly the Omega the
  device generated.
* ``record=``: a list that receives per-block diagnostics (top-2 pivot norm
  gap) so a pivot mismatch can be classified as a near-tie.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# constants (reference.py:40,44; sketch.py:38; randomized.py:56; jacobi.py:20-21)
# ---------------------------------------------------------------------------
NORM_GUARD = 2.0 ** -40
RANK_FLOOR = 2.0 ** -52
SAMPLE_FLOOR = 2.0 ** -48
DIAG_FLOOR = 2.0 ** -52
_JACOBI_SWEEPS = 60
_JACOBI_TOL = 1e-15

# splitmix64 constants (rng.py:32-34)
SM_GOLDEN = 0x9E3779B97F4A7C15
SM_MIX1 = 0xBF58476D1CE4E5B9
SM_MIX2 = 0x94D049BB133111EB
_U64 = (1 << 64) - 1


# ---------------------------------------------------------------------------
# counter-based Gaussian stream (rng.py:38-93)
# ---------------------------------------------------------------------------
def mix_words(seed: int, ctr: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer of seed + (ctr+1)*GOLDEN, mod 2^64 (rng.py:38-42)."""
    g, m1, m2 = np.uint64(SM_GOLDEN), np.uint64(SM_MIX1), np.uint64(SM_MIX2)
    z = np.uint64(seed & _U64) + (ctr + np.uint64(1)) * g
    z = (z ^ (z >> np.uint64(30))) * m1
    z = (z ^ (z >> np.uint64(27))) * m2
    return z ^ (z >> np.uint64(31))


def open_uniforms(seed: int, ctr: np.ndarray) -> np.ndarray:
    """Top 53 bits -> (u + 0.5) 2^-53 in (0, 1) (rng.py:45-46)."""
    return ((mix_words(seed, ctr) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53


def gauss_stream(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """Box-Muller normals at stream positions offset..offset+count-1 (rng.py:49-62).

    Position i pairs with its partner inside the pair floor(i/2); even
    positions take the cosine branch, odd positions the sine branch.
    """
    if count < 0 or offset < 0:
        raise ValueError("count and offset must be nonnegative")
    if count == 0:
        return np.empty(0)
    pos = np.arange(offset, offset + count, dtype=np.uint64)
    base = (pos >> np.uint64(1)) * np.uint64(2)
    u1 = open_uniforms(seed, base)
    u2 = open_uniforms(seed, base + np.uint64(1))
    r = np.sqrt(-2.0 * np.log(u1))
    theta = (2.0 * np.pi) * u2
    return np.where((pos & np.uint64(1)) == 0, r * np.cos(theta), r * np.sin(theta))


def gauss_matrix(rows: int, cols: int, seed: int, offset: int = 0) -> np.ndarray:
    """Column-major fill from the stream (rng.py:65-70)."""
    if rows < 0 or cols < 0:
        raise ValueError("matrix dimensions must be nonnegative")
    flat = gauss_stream(seed, rows * cols, offset=offset)
    return np.asfortranarray(flat.reshape((rows, cols), order="F"))


class GaussStream:
    """Sequential cursor over one seed's stream (rng.py:73-93)."""

    def __init__(self, seed: int):
        self.seed = int(seed) & _U64
        self.position = 0

    def draw(self, count: int) -> np.ndarray:
        out = gauss_stream(self.seed, count, offset=self.position)
        self.position += count
        return out

    def draw_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = gauss_matrix(rows, cols, self.seed, offset=self.position)
        self.position += rows * cols
        return out


# ---------------------------------------------------------------------------
# input contract (validation.py:21-82)
# ---------------------------------------------------------------------------
def as_checked(A, name: str = "A", copy: bool = False) -> np.ndarray:
    M = (np.array(A, dtype=np.float64, order="F", copy=True) if copy
         else np.asfortranarray(A, dtype=np.float64))
    if M.ndim != 2:
        raise ValueError(f"{name} must be 2-dimensional, got ndim={M.ndim}")
    if M.size and not np.isfinite(M).all():
        raise ValueError(f"{name} contains {int(np.count_nonzero(~np.isfinite(M)))} non-finite entries")
    return M


def resolve_rank(m: int, n: int, k) -> int:
    if k is None:
        return min(m, n)
    if not 1 <= k <= min(m, n):
        raise ValueError(f"rank k={k} must satisfy 1 <= k <= min(m, n) = {min(m, n)}")
    return int(k)


def check_kbp(m: int, n: int, k: int, b=None, p=None) -> None:
    if k < 0 or k > min(m, n):
        raise ValueError(f"rank k={k} must satisfy 0 <= k <= min(m, n) = {min(m, n)}")
    if b is not None and b < 1:
        raise ValueError(f"block size b={b} must be >= 1")
    if p is not None and p < 0:
        raise ValueError(f"padding p={p} must be >= 0")


def inverse_perm(perm: np.ndarray) -> np.ndarray:
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0], dtype=perm.dtype)
    return inv


# ---------------------------------------------------------------------------
# communication counters (counters.py:26-44)
# ---------------------------------------------------------------------------
@dataclass
class Counters:
    trailing_passes: int = 0
    blas2_volume: int = 0
    blas3_volume: int = 0

    def passes(self, c: int = 1):
        self.trailing_passes += c

    def vol2(self, e: int):
        self.blas2_volume += int(e)

    def vol3(self, p: int, r: int, q: int):
        self.blas3_volume += int(p) * int(r) * int(q)

    def absorb(self, o: "Counters"):
        self.trailing_passes += o.trailing_passes
        self.blas2_volume += o.blas2_volume
        self.blas3_volume += o.blas3_volume


# ---------------------------------------------------------------------------
# Householder / compact WY (householder.py:28-141)
# ---------------------------------------------------------------------------
def reflector(a: np.ndarray):
    """(y, tau, beta), y[0] = 1, beta = -sign(a0)||a|| (householder.py:28-49)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 1 or a.size == 0:
        raise ValueError("reflector expects a nonempty vector")
    nrm = float(np.linalg.norm(a))
    y = np.zeros_like(a)
    y[0] = 1.0
    if nrm == 0.0:
        return y, 0.0, 0.0
    beta = -(1.0 if a[0] >= 0.0 else -1.0) * nrm
    y[1:] = a[1:] / (a[0] - beta)
    tau = 2.0 / (1.0 + float(y[1:] @ y[1:]))
    return y, tau, beta


def t_factor(Y: np.ndarray, tau: np.ndarray) -> np.ndarray:
    """Forward accumulation of T with I - Y T Y^T = H_1...H_j (householder.py:52-61)."""
    j = Y.shape[1]
    T = np.zeros((j, j))
    G = Y.T @ Y
    for c in range(j):
        T[c, c] = tau[c]
        if c:
            T[:c, c] = -tau[c] * (T[:c, :c] @ G[:c, c])
    return T


@dataclass
class WYBlock:
    """Compact-WY block (householder.py:64-91): Q = I - Y T Y^T."""

    Y: np.ndarray
    tau: np.ndarray
    T: np.ndarray = field(default=None)  # type: ignore[assignment]
    offset: int = 0

    def __post_init__(self):
        self.Y = np.asarray(self.Y, dtype=np.float64)
        self.tau = np.asarray(self.tau, dtype=np.float64)
        if self.Y.ndim != 2 or self.tau.shape != (self.Y.shape[1],):
            raise ValueError("Y must be m x j with one tau per reflector")
        if self.T is None:
            self.T = t_factor(self.Y, self.tau)

    @property
    def m(self) -> int:
        return self.Y.shape[0]

    @property
    def width(self) -> int:
        return self.Y.shape[1]


def compose(b1: WYBlock, b2: WYBlock) -> WYBlock:
    """Q1 Q2 as one block (householder.py:94-104)."""
    if b1.m != b2.m:
        raise ValueError("blocks must act on the same row dimension")
    j1, j2 = b1.width, b2.width
    T = np.zeros((j1 + j2, j1 + j2))
    T[:j1, :j1] = b1.T
    T[j1:, j1:] = b2.T
    T[:j1, j1:] = -b1.T @ (b1.Y.T @ b2.Y) @ b2.T
    return WYBlock(np.hstack([b1.Y, b2.Y]), np.concatenate([b1.tau, b2.tau]), T, offset=b1.offset)


def apply_qt(block: WYBlock, C: np.ndarray) -> np.ndarray:
    if block.width:
        W = block.Y.T @ C
        C -= block.Y @ (block.T.T @ W)
    return C


def apply_q(block: WYBlock, C: np.ndarray) -> np.ndarray:
    if block.width:
        W = block.Y.T @ C
        C -= block.Y @ (block.T @ W)
    return C


def apply_all_qt(blocks, C):
    for blk in blocks:
        apply_qt(blk, C)
    return C


def apply_all_q(blocks, C):
    for blk in reversed(blocks):
        apply_q(blk, C)
    return C


def explicit_q(blocks, m: int, r: int) -> np.ndarray:
    Q = np.zeros((m, r), order="F")
    np.fill_diagonal(Q, 1.0)
    return apply_all_q(blocks, Q)


def compose_all(blocks):
    if not blocks:
        return None
    out = blocks[0]
    for blk in blocks[1:]:
        out = compose(out, blk)
    return out


# ---------------------------------------------------------------------------
# result containers (reference.py:61-99; randomized.py:59-97)
# ---------------------------------------------------------------------------
@dataclass
class Pivoted:
    m: int
    n: int
    blocks: list
    R: np.ndarray
    perm: np.ndarray
    achieved_rank: int
    counters: Counters = field(default_factory=Counters)
    w_t: np.ndarray | None = None  # set for the truncated variant

    def q_columns(self, rank=None):
        r = self.achieved_rank if rank is None else min(rank, self.achieved_rank)
        return explicit_q(self.blocks, self.m, r)

    def apply_q(self, C):
        return apply_all_q(self.blocks, C)

    def reconstruct(self, rank=None):
        r = self.achieved_rank if rank is None else min(rank, self.achieved_rank)
        approx = self.q_columns(r) @ self.R[:r, :]
        return np.asfortranarray(approx[:, inverse_perm(self.perm)])

    def rel_residual(self, A, rank=None) -> float:
        denom = np.linalg.norm(A)
        if denom == 0.0:
            return 0.0
        return float(np.linalg.norm(A - self.reconstruct(rank)) / denom)

    @property
    def r_diag(self):
        r = self.achieved_rank
        return np.abs(np.diag(self.R[:r, :r])) if r else np.zeros(0)


@dataclass
class Tuxv:
    U: WYBlock | None
    X: np.ndarray
    V: WYBlock | None
    sigma_est: np.ndarray
    achieved_rank: int
    counters: Counters
    m: int
    n: int

    def u_columns(self):
        return explicit_q([self.U] if self.U else [], self.m, self.achieved_rank)

    def v_columns(self):
        return explicit_q([self.V] if self.V else [], self.n, self.achieved_rank)

    def reconstruct(self):
        if self.achieved_rank == 0:
            return np.zeros((self.m, self.n), order="F")
        return np.asfortranarray(self.u_columns() @ self.X @ self.v_columns().T)


def _nothing(m, n, counters=None, truncated=False) -> Pivoted:
    return Pivoted(m, n, [], np.zeros((0, n), order="F"), np.arange(n, dtype=np.int64), 0,
                   counters or Counters(),
                   w_t=np.zeros((0, n), order="F") if truncated else None)


# ---------------------------------------------------------------------------
# BLAS-2 QRCP core + blocked QRCP + unpivoted blocked QR (reference.py:47-311)
# ---------------------------------------------------------------------------
def downdate(norms_sq, ref_sq, row, guard: float = NORM_GUARD):
    """Remove one R row from squared trailing norms; flag cancellations (reference.py:47-58)."""
    norms_sq = norms_sq - row * row
    bad = norms_sq < guard * ref_sq
    np.maximum(norms_sq, 0.0, out=norms_sq)
    return norms_sq, bad


def _floor_sq(work: np.ndarray) -> float:
    return (RANK_FLOOR * float(np.linalg.norm(work))) ** 2


def pivoted_core(work: np.ndarray, k: int, cnt: Counters, gaps=None):
    """In-place BLAS-2 QRCP (reference.py:107-150). Returns (taus, perm, achieved).

    ``gaps`` (optional list) receives, per step, the relative gap between the
    largest and second-largest trailing squared norm.
    """
    m, n = work.shape
    steps = min(k, m, n)
    perm = np.arange(n, dtype=np.int64)
    taus = np.zeros(steps)
    nsq = np.einsum("ij,ij->j", work, work)
    rsq = nsq.copy()
    floor_sq = _floor_sq(work)
    done = 0
    for j in range(steps):
        c = j + int(np.argmax(nsq[j:]))
        if gaps is not None:
            tail = np.sort(nsq[j:])[::-1]
            gaps.append(float((tail[0] - tail[1]) / tail[0]) if tail.size > 1 and tail[0] > 0 else 1.0)
        if nsq[c] <= floor_sq:
            break
        if c != j:
            work[:, [j, c]] = work[:, [c, j]]
            perm[[j, c]] = perm[[c, j]]
            nsq[[j, c]] = nsq[[c, j]]
            rsq[[j, c]] = rsq[[c, j]]
        y, tau, beta = reflector(work[j:, j])
        rest = n - j - 1
        if rest:
            w = tau * (y @ work[j:, j + 1:])
            work[j:, j + 1:] -= np.outer(y, w)
            cnt.vol2(2 * (m - j) * rest)
        cnt.passes()
        work[j, j] = beta
        work[j + 1:, j] = y[1:]
        taus[j] = tau
        done = j + 1
        if rest:
            nsq[j + 1:], bad = downdate(nsq[j + 1:], rsq[j + 1:], work[j, j + 1:])
            if bad.any():
                for c2 in (j + 1 + np.nonzero(bad)[0]):
                    v = work[j + 1:, c2]
                    exact = float(v @ v)
                    nsq[c2] = exact
                    rsq[c2] = exact
    return taus[:done], perm, done


def packed_block(work: np.ndarray, taus: np.ndarray, done: int) -> WYBlock:
    """Explicit unit-lower Y from tails packed under the diagonal (reference.py:153-159)."""
    m = work.shape[0]
    Y = np.zeros((m, done), order="F")
    for c in range(done):
        Y[c, c] = 1.0
        Y[c + 1:, c] = work[c + 1:, c]
    return WYBlock(Y, taus)


def qrcp_blas2(A, k=None) -> Pivoted:
    """reference.py:162-171."""
    work = as_checked(A, copy=True)
    m, n = work.shape
    kk = resolve_rank(m, n, k)
    cnt = Counters()
    taus, perm, done = pivoted_core(work, kk, cnt)
    blocks = [packed_block(work, taus, done)] if done else []
    return Pivoted(m, n, blocks, np.triu(work[:done, :]), perm, done, cnt)


def qrcp_blocked(A, k=None, b: int = 32) -> Pivoted:
    """Blocked QRCP with deferred trailing update (reference.py:174-263)."""
    if b < 1:
        raise ValueError("block size b must be >= 1")
    work = as_checked(A, copy=True)
    m, n = work.shape
    kk = resolve_rank(m, n, k)
    cnt = Counters()
    perm = np.arange(n, dtype=np.int64)
    nsq = np.einsum("ij,ij->j", work, work)
    rsq = nsq.copy()
    floor_sq = _floor_sq(work)
    blocks = []
    done = 0
    out_of_rank = False
    while done < kk and not out_of_rank:
        i0 = done
        bb = min(b, kk - i0)
        mr = m - i0
        Yp = np.zeros((mr, bb), order="F")
        Wt = np.zeros((bb, n - i0), order="F")
        tp = np.zeros(bb)
        width = 0
        for t in range(bb):
            j = i0 + t
            c = j + int(np.argmax(nsq[j:]))
            if nsq[c] <= floor_sq:
                out_of_rank = True
                break
            if c != j:
                work[:, [j, c]] = work[:, [c, j]]
                perm[[j, c]] = perm[[c, j]]
                nsq[[j, c]] = nsq[[c, j]]
                rsq[[j, c]] = rsq[[c, j]]
                Wt[:, [t, c - i0]] = Wt[:, [c - i0, t]]
            if t:
                work[j:, j] -= Yp[t:, :t] @ Wt[:t, t]
            y, tau, beta = reflector(work[j:, j])
            Yp[t:, t] = y
            tp[t] = tau
            work[j, j] = beta
            work[j + 1:, j] = y[1:]
            if j + 1 < n:
                yA = y @ work[j:, j + 1:]
                if t:
                    yA -= (y @ Yp[t:, :t]) @ Wt[:t, t + 1:]
                Wt[t, t + 1:] = tau * yA
                cnt.vol2((m - j) * (n - j - 1))
                work[j, j + 1:] -= Yp[t, :t + 1] @ Wt[:t + 1, t + 1:]
            cnt.passes()
            width = t + 1
            done = j + 1
            if j + 1 < n:
                nsq[j + 1:], bad = downdate(nsq[j + 1:], rsq[j + 1:], work[j, j + 1:])
                if bad.any():
                    for c2 in (j + 1 + np.nonzero(bad)[0]):
                        v = work[j + 1:, c2] - Yp[t + 1:, :t + 1] @ Wt[:t + 1, c2 - i0]
                        exact = float(v @ v)
                        nsq[c2] = exact
                        rsq[c2] = exact
        if width == 0:
            break
        Yf = np.zeros((m, width), order="F")
        Yf[i0:, :] = Yp[:, :width]
        blocks.append(WYBlock(Yf, tp[:width].copy(), offset=i0))
        ncols = n - (i0 + width)
        if ncols and mr - width > 0 and not out_of_rank:
            work[i0 + width:, i0 + width:] -= Yp[width:, :width] @ Wt[:width, width:n - i0]
            cnt.passes()
            cnt.vol3(mr - width, width, ncols)
    return Pivoted(m, n, blocks, np.triu(work[:done, :]), perm, done, cnt)


def qr_blocked(A, k=None, b: int = 32) -> Pivoted:
    """Blocked unpivoted Householder QR (reference.py:266-311)."""
    if b < 1:
        raise ValueError("block size b must be >= 1")
    work = as_checked(A, copy=True)
    m, n = work.shape
    kk = resolve_rank(m, n, k)
    cnt = Counters()
    blocks = []
    for i0 in range(0, kk, b):
        bb = min(b, kk - i0)
        tp = np.zeros(bb)
        for t in range(bb):
            j = i0 + t
            y, tau, beta = reflector(work[j:, j])
            tp[t] = tau
            if j + 1 < i0 + bb:
                w = tau * (y @ work[j:, j + 1:i0 + bb])
                work[j:, j + 1:i0 + bb] -= np.outer(y, w)
            work[j, j] = beta
            work[j + 1:, j] = y[1:]
        Yf = np.zeros((m, bb), order="F")
        for t in range(bb):
            Yf[i0 + t, t] = 1.0
            Yf[i0 + t + 1:, t] = work[i0 + t + 1:, i0 + t]
        blk = WYBlock(Yf, tp, offset=i0)
        blocks.append(blk)
        ncols = n - (i0 + bb)
        if ncols:
            Yl = Yf[i0:, :]
            W = blk.T.T @ (Yl.T @ work[i0:, i0 + bb:])
            work[i0:, i0 + bb:] -= Yl @ W
            cnt.passes(2)
            cnt.vol3(bb, m - i0, ncols)
            cnt.vol3(m - i0, bb, ncols)
    return Pivoted(m, n, blocks, np.triu(work[:kk, :]), np.arange(n, dtype=np.int64), kk, cnt)


# ---------------------------------------------------------------------------
# sketch machinery (sketch.py:60-149)
# ---------------------------------------------------------------------------
def sketch(A: np.ndarray, ell: int, stream: GaussStream, cnt: Counters | None = None,
           mid_loop: bool = False, omega: np.ndarray | None = None) -> np.ndarray:
    """B = Omega A (sketch.py:60-76). ``omega`` overrides the stream draw."""
    m, n = A.shape
    if ell < 1:
        raise ValueError("sample must have at least one row")
    Om = stream.draw_matrix(ell, m) if omega is None else np.asarray(omega, dtype=np.float64)
    B = np.asfortranarray(Om @ A)
    if cnt is not None:
        cnt.vol3(ell, m, n)
        if mid_loop:
            cnt.passes()
    return B


@dataclass
class Sample:
    """U^T B P = [S11 S12; 0 S22] after a halted QRCP (sketch.py:79-94)."""

    B: np.ndarray
    S11: np.ndarray
    S12: np.ndarray
    S22: np.ndarray
    local_perm: np.ndarray
    u_block: WYBlock
    achieved: int


def sample_pivots(B: np.ndarray, b: int, gaps=None) -> Sample:
    """Halted QRCP of the sample (sketch.py:97-119)."""
    work = as_checked(B, copy=True)
    ell, n = work.shape
    if not 0 <= b <= min(ell, n):
        raise ValueError(f"need 0 <= b <= min(l, n) = {min(ell, n)}, got b={b}")
    taus, perm, done = pivoted_core(work, b, Counters(), gaps)
    return Sample(work, np.triu(work[:done, :done]), work[:done, done:], work[done:, done:],
                  perm, packed_block(work, taus, done), done)


def back_solve(R11: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """Row-oriented back substitution X = R11^-1 rhs (sketch.py:122-129)."""
    X = np.array(rhs, dtype=np.float64, order="F", copy=True)
    nb = R11.shape[0]
    for i in range(nb - 1, -1, -1):
        if i + 1 < nb:
            X[i] -= R11[i, i + 1:] @ X[i + 1:]
        X[i] /= R11[i, i]
    return X


def sample_refresh(st: Sample, R11: np.ndarray, R12: np.ndarray) -> np.ndarray:
    """B_next = [S12 - S11 R11^-1 R12; S22] (sketch.py:132-149)."""
    bh = st.achieved
    if R11.shape != (bh, bh) or R12.shape[0] != bh:
        raise ValueError("R11/R12 do not match the sample's achieved block size")
    d = np.abs(np.diag(R11))
    if bh and d.min() <= 2.0 ** -52 * d[0]:
        raise np.linalg.LinAlgError("R11 is numerically singular; the factorization rank is exhausted")
    X = back_solve(R11, R12)
    return np.asfortranarray(np.vstack([st.S12 - st.S11 @ X, st.S22]))


# ---------------------------------------------------------------------------
# randomized drivers (randomized.py:107-406)
# ---------------------------------------------------------------------------
def panel_factor(work: np.ndarray, i0: int, bb: int):
    """Unpivoted DGEQR2-style panel on work[i0:, i0:i0+bb]; stops at beta == 0
    (randomized.py:107-130). Returns (Ypan, taus, completed)."""
    m = work.shape[0]
    Yp = np.zeros((m - i0, bb), order="F")
    tp = np.zeros(bb)
    done = 0
    for t in range(bb):
        j = i0 + t
        y, tau, beta = reflector(work[j:, j])
        if beta == 0.0:
            break
        if t + 1 < bb:
            w = tau * (y @ work[j:, j + 1:i0 + bb])
            work[j:, j + 1:i0 + bb] -= np.outer(y, w)
        work[j, j] = beta
        work[j + 1:, j] = y[1:]
        Yp[t:, t] = y
        tp[t] = tau
        done = t + 1
    return Yp[:, :done], tp[:done], done


def r11_usable(R11: np.ndarray) -> bool:
    """randomized.py:133-135."""
    d = np.abs(np.diag(R11))
    return d.size > 0 and d.min() > DIAG_FLOOR * d[0]


def sample_floor_sq(B: np.ndarray) -> float:
    """randomized.py:138-140."""
    top = np.einsum("ij,ij->j", B, B).max() if B.size else 0.0
    return SAMPLE_FLOOR ** 2 * top


def ssrqrcp(A, k: int, p: int = 8, seed: int = 0, omega=None) -> Pivoted:
    """Single-sample randomized QRCP (randomized.py:143-163)."""
    A = as_checked(A)
    m, n = A.shape
    check_kbp(m, n, k, None, p)
    if k == 0:
        return _nothing(m, n)
    ell = k + p
    if ell >= m:
        return qrcp_blocked(A, k, b=min(32, k))
    cnt = Counters()
    B = sketch(A, ell, GaussStream(seed), cnt, omega=omega)
    st = sample_pivots(B, k)
    if st.achieved == 0:
        return _nothing(m, n, cnt)
    qf = qr_blocked(np.asfortranarray(A[:, st.local_perm]), st.achieved, b=min(32, st.achieved))
    cnt.absorb(qf.counters)
    return Pivoted(m, n, qf.blocks, qf.R, st.local_perm.copy(), st.achieved, cnt)


def _blocked_randomized(A, k, b, p, seed, resample, omega=None, record=None) -> Pivoted:
    """RQRCP / RSRQRCP driver (randomized.py:166-224)."""
    A = as_checked(A)
    m, n = A.shape
    check_kbp(m, n, k, b, p)
    if k == 0:
        return _nothing(m, n)
    ell = b + p
    if ell >= m:
        return qrcp_blocked(A, k, b)
    cnt = Counters()
    stream = GaussStream(seed)
    work = np.array(A, dtype=np.float64, order="F", copy=True)
    perm = np.arange(n, dtype=np.int64)
    B = sketch(work, ell, stream, cnt, omega=omega)
    floor_sq = sample_floor_sq(B)
    blocks = []
    done = 0
    while done < k:
        i0 = done
        bb = min(b, k - i0)
        csq = np.einsum("ij,ij->j", B, B)
        if csq.size == 0 or csq.max() <= floor_sq:
            break
        gaps = [] if record is not None else None
        st = sample_pivots(B, bb, gaps)
        if record is not None:
            record.append({"i0": i0, "gaps": gaps, "local_perm": st.local_perm.copy()})
        if st.achieved == 0:
            break
        work[:, i0:] = work[:, i0:][:, st.local_perm]
        perm[i0:] = perm[i0:][st.local_perm]
        Yp, tp, bh = panel_factor(work, i0, st.achieved)
        if bh == 0:
            break
        Yf = np.zeros((m, bh), order="F")
        Yf[i0:, :] = Yp
        blk = WYBlock(Yf, tp.copy(), offset=i0)
        blocks.append(blk)
        ncols = n - (i0 + bh)
        if ncols:
            W = blk.T.T @ (Yp.T @ work[i0:, i0 + bh:])
            work[i0:, i0 + bh:] -= Yp @ W
            cnt.passes(2)
            cnt.vol3(bh, m - i0, ncols)
            cnt.vol3(m - i0, bh, ncols)
        done = i0 + bh
        if bh < bb or done >= k or ncols == 0:
            break
        if resample:
            B = sketch(work[done:, done:], ell, stream, cnt, mid_loop=True)
        else:
            R11 = np.triu(work[i0:done, i0:done])
            if not r11_usable(R11):
                break
            B = sample_refresh(st, R11, work[i0:done, done:])
    return Pivoted(m, n, blocks, np.triu(work[:done, :]), perm, done, cnt)


def rqrcp(A, k: int, b: int = 32, p: int = 8, seed: int = 0, omega=None, record=None) -> Pivoted:
    """randomized.py:227-229."""
    return _blocked_randomized(A, k, b, p, seed, False, omega, record)


def rsrqrcp(A, k: int, b: int = 32, p: int = 8, seed: int = 0) -> Pivoted:
    """randomized.py:232-234."""
    return _blocked_randomized(A, k, b, p, seed, True)


def _truncated_fallback(pf: Pivoted, A: np.ndarray) -> Pivoted:
    """Dense w_t for the l >= m fallback (randomized.py:237-247)."""
    w_t = np.zeros((pf.achieved_rank, pf.n), order="F")
    if pf.blocks:
        allb = compose_all(pf.blocks)
        w_t = allb.T.T @ (allb.Y.T @ A[:, pf.perm])
    return Pivoted(pf.m, pf.n, pf.blocks, pf.R, pf.perm, pf.achieved_rank, pf.counters, w_t=w_t)


def trqrcp(A, k: int, b: int = 32, p: int = 8, seed: int = 0, allow_large_k: bool = False,
           omega=None, record=None) -> Pivoted:
    """Truncated RQRCP without trailing update (randomized.py:250-341)."""
    A = as_checked(A)
    m, n = A.shape
    check_kbp(m, n, k, b, p)
    if not allow_large_k and k > min(m, n) // 2:
        raise ValueError("trqrcp targets k <= min(m, n)/2; pass allow_large_k=True to override")
    if k == 0:
        return _nothing(m, n, truncated=True)
    ell = b + p
    if ell >= m:
        return _truncated_fallback(qrcp_blocked(A, k, b), A)
    cnt = Counters()
    stream = GaussStream(seed)
    work = np.array(A, dtype=np.float64, order="F", copy=True)
    perm = np.arange(n, dtype=np.int64)
    B = sketch(work, ell, stream, cnt, omega=omega)
    floor_sq = sample_floor_sq(B)
    Yg = np.zeros((m, k), order="F")
    Wg = np.zeros((k, n), order="F")
    Rg = np.zeros((k, n), order="F")
    blocks = []
    done = 0
    while done < k:
        i0 = done
        bb = min(b, k - i0)
        csq = np.einsum("ij,ij->j", B, B)
        if csq.size == 0 or csq.max() <= floor_sq:
            break
        gaps = [] if record is not None else None
        st = sample_pivots(B, bb, gaps)
        if record is not None:
            record.append({"i0": i0, "gaps": gaps, "local_perm": st.local_perm.copy()})
        if st.achieved == 0:
            break
        lp = st.local_perm
        work[:, i0:] = work[:, i0:][:, lp]
        perm[i0:] = perm[i0:][lp]
        Wg[:, i0:] = Wg[:, i0:][:, lp]
        Rg[:, i0:] = Rg[:, i0:][:, lp]
        panel = np.array(work[i0:, i0:i0 + st.achieved], order="F", copy=True)
        if i0:
            panel -= Yg[i0:, :i0] @ Wg[:i0, i0:i0 + st.achieved]
        Yp, tp, bh = panel_factor(panel, 0, st.achieved)
        if bh == 0:
            break
        R11 = np.triu(panel[:bh, :bh])
        T2 = t_factor(Yp, tp)
        Yg[i0:, i0:i0 + bh] = Yp
        Yf = np.zeros((m, bh), order="F")
        Yf[i0:, :] = Yp
        blocks.append(WYBlock(Yf, tp.copy(), T2, offset=i0))
        Rg[i0:i0 + bh, i0:i0 + bh] = R11
        ntr = n - (i0 + bh)
        R12 = np.zeros((bh, 0))
        if ntr:
            tc = slice(i0 + bh, n)
            G = Yp.T @ work[i0:, tc]
            cnt.passes()
            cnt.vol3(bh, m - i0, ntr)
            if i0:
                G -= (Yp.T @ Yg[i0:, :i0]) @ Wg[:i0, tc]
            Wg[i0:i0 + bh, tc] = T2.T @ G
            R12 = work[i0:i0 + bh, tc] - Yg[i0:i0 + bh, :i0 + bh] @ Wg[:i0 + bh, tc]
            Rg[i0:i0 + bh, tc] = R12
        done = i0 + bh
        if bh < bb or done >= k or ntr == 0:
            break
        if not r11_usable(R11):
            break
        B = sample_refresh(st, R11, R12)
    return Pivoted(m, n, blocks, np.asfortranarray(np.triu(Rg[:done, :])), perm, done, cnt,
                   w_t=np.asfortranarray(Wg[:done, :]))


def tuxv(A, k: int, j_max: int = 1, b: int = 32, p: int = 8, seed: int = 0,
         refine_sigma: bool = False, allow_large_k: bool = False, omega=None) -> Tuxv:
    """TRQRCP + QLP flip-flop passes (randomized.py:353-406)."""
    A = as_checked(A)
    m, n = A.shape
    if j_max < 1:
        raise ValueError("j_max must be >= 1")
    tf = trqrcp(A, k, b=b, p=p, seed=seed, allow_large_k=allow_large_k, omega=omega)
    kh = tf.achieved_rank
    cnt = tf.counters
    if kh == 0:
        return Tuxv(None, np.zeros((0, 0)), None, np.zeros(0), 0, cnt, m, n)
    Z0 = tf.R[:, inverse_perm(tf.perm)]
    vf = qr_blocked(np.asfortranarray(Z0.T), kh, b)
    cnt.absorb(vf.counters)
    vb, ub = vf.blocks, []
    X = np.asfortranarray(vf.R[:kh, :kh].T)
    for j in range(1, j_max + 1):
        if j % 2 == 1:
            Z = np.asfortranarray(A @ explicit_q(vb, n, kh))
            cnt.passes()
            cnt.vol3(m, n, kh)
            uf = qr_blocked(Z, kh, b)
            cnt.absorb(uf.counters)
            ub = uf.blocks
            X = uf.R[:kh, :kh]
        else:
            Z = np.asfortranarray((explicit_q(ub, m, kh).T @ A).T)
            cnt.passes()
            cnt.vol3(kh, m, n)
            vf = qr_blocked(Z, kh, b)
            cnt.absorb(vf.counters)
            vb = vf.blocks
            X = np.asfortranarray(vf.R[:kh, :kh].T)
    sig = np.abs(np.diag(X))
    if refine_sigma:
        sig = jacobi_svd(X)[1]
    return Tuxv(compose_all(ub), X, compose_all(vb), sig, kh, cnt, m, n)


# ---------------------------------------------------------------------------
# one-sided Jacobi SVD for refine_sigma (jacobi.py:24-117)
# ---------------------------------------------------------------------------
def _tournament(n: int):
    seats = list(range(n)) + ([] if n % 2 == 0 else [-1])
    q = len(seats)
    out = []
    for _ in range(q - 1):
        prs = [(seats[i], seats[q - 1 - i]) for i in range(q // 2)
               if seats[i] >= 0 and seats[q - 1 - i] >= 0]
        out.append((np.array([a for a, _ in prs]), np.array([c for _, c in prs])))
        seats = [seats[0], seats[-1]] + seats[1:-1]
    return out


def jacobi_svd(A):
    """Hestenes one-sided Jacobi (jacobi.py:50-117): (U, sigma, V)."""
    A = as_checked(A, copy=True)
    m, n = A.shape
    if min(m, n) > 4096:
        raise ValueError("jacobi_svd targets desk-scale matrices (min dim <= 4096)")
    if m < n:
        V, s, U = jacobi_svd(A.T)
        return U, s, V
    if n == 0:
        return np.zeros((m, 0)), np.zeros(0), np.zeros((0, 0))
    W = A
    V = np.eye(n, order="F")
    if np.linalg.norm(W) == 0.0:
        return np.eye(m, n), np.zeros(n), np.eye(n)
    sched = _tournament(n)
    for _ in range(_JACOBI_SWEEPS):
        moved = False
        for ii, jj in sched:
            Wi, Wj = W[:, ii], W[:, jj]
            al = np.einsum("ij,ij->j", Wi, Wi)
            be = np.einsum("ij,ij->j", Wj, Wj)
            ga = np.einsum("ij,ij->j", Wi, Wj)
            live = np.abs(ga) > _JACOBI_TOL * np.sqrt(al * be)
            if not live.any():
                continue
            moved = True
            ii, jj = ii[live], jj[live]
            a, bq, g = al[live], be[live], ga[live]
            zeta = (bq - a) / (2.0 * g)
            t = np.sign(zeta) / (np.abs(zeta) + np.sqrt(1.0 + zeta * zeta))
            t[zeta == 0.0] = 1.0
            c = 1.0 / np.sqrt(1.0 + t * t)
            s = c * t
            Wi, Wj = W[:, ii].copy(), W[:, jj]
            W[:, ii] = c * Wi - s * Wj
            W[:, jj] = s * Wi + c * Wj
            Vi, Vj = V[:, ii].copy(), V[:, jj]
            V[:, ii] = c * Vi - s * Vj
            V[:, jj] = s * Vi + c * Vj
        if not moved:
            break
    else:
        raise np.linalg.LinAlgError("Jacobi sweeps did not converge")
    sig = np.linalg.norm(W, axis=0)
    order = np.argsort(-sig, kind="stable")
    sig, W, V = sig[order], W[:, order], V[:, order]
    U = np.zeros((m, n), order="F")
    r = int(np.count_nonzero(sig > sig[0] * m * np.finfo(np.float64).eps))
    if r:
        U[:, :r] = W[:, :r] / sig[:r]
    if r < n:
        U[:, r:n] = np.linalg.qr(U[:, :r], mode="complete")[0][:, r:n]
    return U, sig, V


# ---------------------------------------------------------------------------
# synthetic inputs (synth.py:12-40)
# ---------------------------------------------------------------------------
def synth_decay(m: int, n: int, ratio: float = 0.8, seed: int = 0) -> np.ndarray:
    if not 0.0 < ratio < 1.0:
        raise ValueError("decay ratio must lie in (0, 1)")
    kk = min(m, n)
    st = GaussStream(seed)
    U, _ = np.linalg.qr(st.draw_matrix(m, kk))
    V, _ = np.linalg.qr(st.draw_matrix(n, kk))
    return np.asfortranarray((U * ratio ** np.arange(kk)) @ V.T)


def synth_kahan(n: int, c: float = 0.285) -> np.ndarray:
    s = np.sqrt(1.0 - c * c)
    K = np.eye(n) - c * np.triu(np.ones((n, n)), 1)
    K *= (s ** np.arange(n))[:, None]
    return np.asfortranarray(K)


__all__ = [name for name in dir() if not name.startswith("_") and name not in ("annotations", "math")]

"""Communication counters carried by every result (reference: counters.py:26-44).

The reference charges its analytic model while it runs; the GPU drivers run
with no host synchronisation, so the same numbers are derived afterwards from
the loop's final state (achieved rank, block count, stop reason).  The
formulas are the reference's own charge sites, cited per function.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class CommCounters:
    trailing_passes: int = 0
    blas2_volume: int = 0
    blas3_volume: int = 0

    def add_pass(self, count: int = 1) -> None:
        self.trailing_passes += count

    def add_blas2(self, elements: int) -> None:
        self.blas2_volume += int(elements)

    def add_blas3(self, p: int, r: int, q: int) -> None:
        self.blas3_volume += int(p) * int(r) * int(q)

    def merge(self, other: "CommCounters") -> None:
        self.trailing_passes += other.trailing_passes
        self.blas2_volume += other.blas2_volume
        self.blas3_volume += other.blas3_volume


# stop reasons that fire at the END of a completed block (randomized.py:212-213)
END_OF_BLOCK_STOPS = {1, 5, 6}


def block_widths(achieved: int, nblocks: int, b: int):
    """(i0, width) of every completed block: all full except possibly the last."""
    out = []
    for J in range(nblocks):
        i0 = J * b
        out.append((i0, min(b, achieved - i0)))
    return out


def rqrcp_counters(m, n, b, ell, achieved, nblocks, reason, resample) -> CommCounters:
    """randomized.py:208-210 per block, sketch.py:72-75 per sketch."""
    c = CommCounters()
    c.add_blas3(ell, m, n)
    for i0, bh in block_widths(achieved, nblocks, b):
        ncols = n - (i0 + bh)
        if ncols:
            c.add_pass(2)
            c.add_blas3(bh, m - i0, ncols)
            c.add_blas3(m - i0, bh, ncols)
    if resample:
        nres = nblocks - (1 if (nblocks and reason in END_OF_BLOCK_STOPS) else 0)
        for J in range(nres):
            a = (J + 1) * b
            c.add_blas3(ell, m - a, n - a)
            c.add_pass()
    return c


def trqrcp_counters(m, n, b, ell, achieved, nblocks) -> CommCounters:
    """randomized.py:323-324 per block plus the sketch."""
    c = CommCounters()
    c.add_blas3(ell, m, n)
    for i0, bh in block_widths(achieved, nblocks, b):
        nt = n - (i0 + bh)
        if nt:
            c.add_pass()
            c.add_blas3(bh, m - i0, nt)
    return c


def qr_blocked_counters(m, n, k, b) -> CommCounters:
    """reference.py:303-307."""
    c = CommCounters()
    for i0 in range(0, k, b):
        bb = min(b, k - i0)
        ncols = n - (i0 + bb)
        if ncols:
            c.add_pass(2)
            c.add_blas3(bb, m - i0, ncols)
            c.add_blas3(m - i0, bb, ncols)
    return c


def qrcp_blocked_counters(m, n, kmax, b, achieved) -> CommCounters:
    """reference.py:222-252: one pass + blas2 per pivot, one GEMM pass per block."""
    c = CommCounters()
    exhausted = achieved < kmax
    for j in range(achieved):
        if j + 1 < n:
            c.add_blas2((m - j) * (n - j - 1))
        c.add_pass()
    i0 = 0
    while i0 < achieved:
        jj = min(b, achieved - i0)
        last = i0 + jj >= achieved
        ncols = n - (i0 + jj)
        # exhaustion inside this (last) block suppresses its GEMM (reference.py:249)
        if ncols and (m - i0) - jj > 0 and not (last and exhausted and achieved % b != 0):
            c.add_pass()
            c.add_blas3((m - i0) - jj, jj, ncols)
        i0 += jj
    return c


def qrcp_blas2_counters(m, n, achieved) -> CommCounters:
    """reference.py:131-136."""
    c = CommCounters()
    for j in range(achieved):
        ntrail = n - j - 1
        if ntrail:
            c.add_blas2(2 * (m - j) * ntrail)
        c.add_pass()
    return c

"""Inputs of BASELINE.json's configs C2-C5, generated on the HOST exactly as the
reference builds them, in parallel.

The Gaussian stream is the reference's counter-based recipe (rng.py:38-70); a
rows x cols column-major matrix drawn at stream offset `off` is the column
slice [j0, j1) = normals(seed, rows*(j1-j0), off + j0*rows), so column chunks
can be drawn by independent worker processes and the bytes are identical to
one big `giid` call.  The draw function is passed in: make_golden*.py uses the
REAL reference (sketchqr.rng.normals) and the GPU tests the oracle
restatement (oracle.port.gauss_stream, bit-identical, tests/test_oracle.py).

`column_digest` hashes the F-order bytes chunk by chunk (sha256), so a GPU box
whose NumPy SIMD transcendentals differ from this container's is detected.

Test infrastructure only (not part of the product package).
"""
from __future__ import annotations

import hashlib
import multiprocessing as mp
import os

import numpy as np

_CHUNK_ELEMS = 1 << 24          # normals per worker task (~128 MB of fp64)


def _worker_draw(args):
    draw, shm_name, shape, rows, seed, off, j0, j1, scale = args
    from multiprocessing import shared_memory
    shm = shared_memory.SharedMemory(name=shm_name)
    try:
        out = np.ndarray(shape, dtype=np.float64, buffer=shm.buf, order="F")
        v = draw(seed, rows * (j1 - j0), off + j0 * rows).reshape((rows, j1 - j0), order="F")
        if scale != 1.0:
            v = v * scale
        out[:, j0:j1] = v
    finally:
        shm.close()
    return j1 - j0


def parallel_giid(draw, rows: int, cols: int, seed: int, offset: int = 0, scale: float = 1.0,
                  procs: int | None = None) -> np.ndarray:
    """scale * giid(rows, cols, seed, offset), drawn by a process pool into shared memory."""
    from multiprocessing import shared_memory
    procs = procs or max(1, min(os.cpu_count() or 1, 32))
    nbytes = max(8, rows * cols * 8)
    shm = shared_memory.SharedMemory(create=True, size=nbytes)
    try:
        step = max(1, _CHUNK_ELEMS // max(rows, 1))
        tasks = [(draw, shm.name, (rows, cols), rows, seed, offset, j0, min(cols, j0 + step), scale)
                 for j0 in range(0, cols, step)]
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            for _ in pool.imap_unordered(_worker_draw, tasks):
                pass
        view = np.ndarray((rows, cols), dtype=np.float64, buffer=shm.buf, order="F")
        out = np.empty((rows, cols), dtype=np.float64, order="F")
        out[...] = view
        del view
    finally:
        shm.close()
        shm.unlink()
    return out


def column_digest(A: np.ndarray, chunk_cols: int = 1024) -> str:
    """sha256 of the column-major bytes of A."""
    h = hashlib.sha256()
    A = np.asfortranarray(A)
    for j0 in range(0, A.shape[1], chunk_cols):
        h.update(np.ascontiguousarray(A[:, j0:j0 + chunk_cols].T).tobytes())
    return h.hexdigest()


def c3_matrix(draw, procs=None) -> np.ndarray:
    """C3: giid(100000, 2000, seed=3)."""
    return parallel_giid(draw, 100000, 2000, 3, procs=procs)


def c4_matrix(draw, procs=None) -> np.ndarray:
    """C4: S = G1 G2^T / ||G1 G2^T||_F with G1 = giid(20000,100,41), G2 = giid(20000,100,42);
    A = S + 1e-6 giid(20000, 20000, seed=43) (BASELINE.json configs[3])."""
    n = 20000
    G1 = parallel_giid(draw, n, 100, 41, procs=1)
    G2 = parallel_giid(draw, n, 100, 42, procs=1)
    A = parallel_giid(draw, n, n, 43, scale=1e-6, procs=procs)
    S = G1 @ G2.T
    S /= np.linalg.norm(S)
    A += S
    return A


def c5_matrix(draw, procs=None) -> np.ndarray:
    """C5: giid(32768, 32768, seed=5)."""
    return parallel_giid(draw, 32768, 32768, 5, procs=procs)

"""Counter-based Gaussian stream of the reference (rng.py:32-93).

``device_giid`` draws on the GPU (libsqr's sqr_gaussian: bit-exact integer
stage, CUDA libm for log/sin/cos).  ``giid`` / ``normals`` / ``NormalStream``
are the host recipe, kept for the bit-identical ``omega="host"`` mode and
for generating inputs exactly as the reference does.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _lib
from ._dev import ColMajor, require_cuda, stream_handle

GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
_M64 = (1 << 64) - 1


def _words(seed: int, ctr: np.ndarray) -> np.ndarray:
    z = np.uint64(seed & _M64) + (ctr + np.uint64(1)) * np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
    return z ^ (z >> np.uint64(31))


def normals(seed: int, count: int, offset: int = 0) -> np.ndarray:
    if count < 0 or offset < 0:
        raise ValueError("count and offset must be nonnegative")
    if count == 0:
        return np.empty(0)
    idx = np.arange(offset, offset + count, dtype=np.uint64)
    even = (idx >> np.uint64(1)) << np.uint64(1)
    u1 = ((_words(seed, even) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    u2 = ((_words(seed, even + np.uint64(1)) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = (2.0 * np.pi) * u2
    return np.where((idx & np.uint64(1)) == 0, rad * np.cos(ang), rad * np.sin(ang))


def giid(rows: int, cols: int, seed: int, offset: int = 0) -> np.ndarray:
    if rows < 0 or cols < 0:
        raise ValueError("matrix dimensions must be nonnegative")
    return np.asfortranarray(normals(seed, rows * cols, offset).reshape((rows, cols), order="F"))


class NormalStream:
    def __init__(self, seed: int):
        self.seed = int(seed) & _M64
        self.position = 0

    def normals(self, count: int) -> np.ndarray:
        out = normals(self.seed, count, self.position)
        self.position += count
        return out

    def matrix(self, rows: int, cols: int) -> np.ndarray:
        out = giid(rows, cols, self.seed, self.position)
        self.position += rows * cols
        return out


_CHUNK = 1 << 18


def host_omega(ell: int, m: int, seed: int, threads: int | None = None) -> np.ndarray:
    """The reference's first draw of every sketch: NormalStream(seed).matrix(l, m),
    bit-identical, drawn by host threads in contiguous counter ranges (NumPy's
    ufuncs release the GIL; each entry depends only on its counter)."""
    total = ell * m
    threads = threads or min(16, os.cpu_count() or 1)
    if total <= 2 * _CHUNK or threads <= 1:
        return giid(ell, m, seed, 0)
    flat = np.empty(total, dtype=np.float64)

    def fill(c0):
        c1 = min(total, c0 + _CHUNK)
        flat[c0:c1] = normals(seed, c1 - c0, c0)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(fill, range(0, total, _CHUNK)))
    return np.asfortranarray(flat.reshape((ell, m), order="F"))


def device_giid(rows: int, cols: int, seed: int, offset: int = 0, transpose: bool = False,
                device=None) -> torch.Tensor:
    """rows x cols Gaussian matrix (or its transpose) generated on the GPU."""
    dev = require_cuda(device)
    r, c = (cols, rows) if transpose else (rows, cols)
    out = ColMajor.empty(r, c, dev)
    _lib.check(_lib.lib().sqr_gaussian(out.ptr, out.ld, rows, cols, int(seed) & _M64, int(offset),
                                       1 if transpose else 0, stream_handle()), "sqr_gaussian")
    return out.view()

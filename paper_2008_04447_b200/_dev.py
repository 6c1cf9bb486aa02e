"""Device plumbing: torch tensors as column-major fp64 storage, workspaces, streams.

torch provides device memory, the current stream and (for multi-GPU)
torch.distributed; every floating-point operation of the factorizations runs
in libsqr's kernels.  There is no CPU path: without a CUDA device these
helpers raise.
"""
from __future__ import annotations

import contextlib
import os
import threading

import numpy as np
import torch

from . import _lib


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2008_04447_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise RuntimeError(f"device {dev} is not a CUDA device")
    return dev


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def even(x: int) -> int:
    return x + (x & 1)


class ColMajor:
    """An m x n fp64 column-major matrix stored as a torch tensor of shape (n, ld)."""

    __slots__ = ("t", "m", "n", "ld")

    def __init__(self, t: torch.Tensor, m: int, n: int, ld: int):
        self.t, self.m, self.n, self.ld = t, m, n, ld

    @classmethod
    def empty(cls, m: int, n: int, device, zero: bool = False, ld: int | None = None) -> "ColMajor":
        ld = even(max(m, 1)) if ld is None else ld
        alloc = torch.zeros if zero else torch.empty
        return cls(alloc((max(n, 1), ld), dtype=torch.float64, device=device), m, n, ld)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def col_ptr(self, row: int, col: int) -> int:
        return self.t.data_ptr() + 8 * (col * self.ld + row)

    def view(self) -> torch.Tensor:
        """m x n logical matrix (a transposed, strided view)."""
        return self.t[: self.n, : self.m].T

    def numpy(self) -> np.ndarray:
        return np.asfortranarray(self.view().cpu().numpy())


_STAGE_BYTES = 64 << 20          # pinned staging chunk of the pipelined upload
_PIPELINE_MIN = 32 << 20         # below this a plain copy is as fast
_staging: dict = {}
_staging_lock = threading.Lock()


def _stagers(device):
    """Two pinned staging buffers + their "free" events, one pair per device."""
    key = str(device)
    with _staging_lock:
        st = _staging.get(key)
        if st is None:
            bufs = [torch.empty(_STAGE_BYTES, dtype=torch.uint8).pin_memory() for _ in range(2)]
            st = _staging[key] = (bufs, threading.Lock())
        return st


def _h2d_pipelined(src: np.ndarray, dst: torch.Tensor) -> None:
    """dst (contiguous CUDA tensor) <- src (contiguous pageable host array, same
    bytes): host threads copy 64 MB chunks into two pinned staging buffers while
    the copy engine moves the previous chunk, so a pageable input crosses
    PCIe at pinned-memory speed instead of through the driver's pageable path."""
    from concurrent.futures import ThreadPoolExecutor
    sb = src.reshape(-1).view(np.uint8)
    db = dst.view(-1).view(torch.uint8)
    total = sb.size
    (bufs, lock) = _stagers(dst.device)
    stream = torch.cuda.current_stream(dst.device)
    events = [None, None]
    nthr = max(1, min(16, (os.cpu_count() or 1)))
    with lock, ThreadPoolExecutor(nthr) as ex:
        for i, c0 in enumerate(range(0, total, _STAGE_BYTES)):
            c1 = min(total, c0 + _STAGE_BYTES)
            k = i & 1
            if events[k] is not None:
                events[k].synchronize()             # the buffer's previous chunk has left
            stage = bufs[k].numpy()
            step = -(-(c1 - c0) // nthr)
            list(ex.map(lambda j: np.copyto(stage[j:min(c1 - c0, j + step)], sb[c0 + j:min(c1, c0 + j + step)]),
                        range(0, c1 - c0, step)))
            db[c0:c1].copy_(bufs[k][:c1 - c0], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            events[k] = ev
        for ev in events:
            if ev is not None:
                ev.synchronize()


def _is_pinned(arr: np.ndarray) -> bool:
    try:
        return torch.from_numpy(arr).is_pinned()
    except Exception:
        return False


def upload(A, device, copy: bool = True) -> ColMajor:
    """Copy a 2-D numpy array / torch tensor into fresh column-major device storage."""
    if isinstance(A, torch.Tensor):
        src = A.detach()
        if src.dim() != 2:
            raise ValueError(f"A must be 2-dimensional, got ndim={src.dim()}")
        m, n = src.shape
        out = ColMajor.empty(m, n, device)
        if m and n:
            out.view().copy_(src.to(device=device, dtype=torch.float64))
        return out
    arr = np.asarray(A)
    if arr.ndim != 2:
        raise ValueError(f"A must be 2-dimensional, got ndim={arr.ndim}")
    m, n = arr.shape
    big = arr.dtype == np.float64 and arr.nbytes >= _PIPELINE_MIN and not _is_pinned(arr)
    if big and arr.flags.c_contiguous and not arr.flags.f_contiguous:
        # C-ordered host input: rows up as they are, transposed on the device
        rows = torch.empty((m, n), dtype=torch.float64, device=device)
        _h2d_pipelined(arr, rows)
        out = ColMajor.empty(m, n, device)
        out.view().copy_(rows)
        return out
    arr = np.asfortranarray(arr, dtype=np.float64)
    out = ColMajor.empty(m, n, device)
    if m and n:
        host = torch.from_numpy(arr.T)  # (n, m) C-contiguous view of the Fortran array
        if big:
            if out.ld == m:
                _h2d_pipelined(arr.T, out.t[:n])
            else:
                tmp = torch.empty((n, m), dtype=torch.float64, device=device)
                _h2d_pipelined(arr.T, tmp)
                out.t[:n, :m].copy_(tmp)
        elif out.ld == m:
            out.t[:n].copy_(host, non_blocking=False)
        else:
            out.t[:n, :m].copy_(host)
    return out


def _copy_check(src_ptr: int, lds: int, m: int, n: int, dst: "ColMajor | None", device) -> int:
    """libsqr copy_check_kernel: optional copy + non-finite count in one read."""
    cnt = torch.zeros(1, dtype=torch.int64, device=device)
    _lib.check(_lib.lib().sqr_copy_check(src_ptr, lds, m, n, dst.ptr if dst is not None else None,
                                         dst.ld if dst is not None else 0, cnt.data_ptr(), stream_handle()),
               "sqr_copy_check")
    return int(cnt.item())


def _device_colmajor(A, device) -> int | None:
    """Leading dimension if A is an fp64 CUDA tensor on `device` in column-major
    layout (stride (1, ld)), else None."""
    if (isinstance(A, torch.Tensor) and A.is_cuda and A.device == torch.device(device) and A.dtype == torch.float64
            and A.dim() == 2 and A.shape[0] > 0 and A.shape[1] > 0 and A.stride(0) == 1
            and A.stride(1) >= A.shape[0]):
        return int(A.stride(1))
    return None


def _device_rowmajor(A, device) -> int | None:
    """Row stride if A is an fp64 CUDA tensor on `device` in row-major layout."""
    if (isinstance(A, torch.Tensor) and A.is_cuda and A.device == torch.device(device) and A.dtype == torch.float64
            and A.dim() == 2 and A.shape[0] > 0 and A.shape[1] > 0 and A.stride(1) == 1
            and A.stride(0) >= A.shape[1]):
        return int(A.stride(0))
    return None


def load_checked(A, device, copy: bool = True, check: bool = True) -> ColMajor:
    """The input contract of validation.check_matrix (validation.py:21-37) on
    the device: 2-D, finite, copied into fresh column-major storage (or, with
    copy=False and a column-major fp64 device input, wrapped read-only).  A
    column-major device input is copied and scanned in ONE pass."""
    lds = _device_colmajor(A, device)
    rls = _device_rowmajor(A, device) if lds is None else None
    if rls is not None:
        # C-ordered device input: tiled transpose + scan in one pass
        m, n = A.shape
        M = ColMajor.empty(m, n, device)
        cnt = torch.zeros(1, dtype=torch.int64, device=device)
        _lib.check(_lib.lib().sqr_copy_check_t(A.data_ptr(), rls, m, n, M.ptr, M.ld, cnt.data_ptr(), stream_handle()),
                   "sqr_copy_check_t")
        bad = int(cnt.item()) if check else 0
    elif lds is not None:
        m, n = A.shape
        if copy:
            M = ColMajor.empty(m, n, device)
        else:
            M = ColMajor(A.as_strided((n, m), (lds, 1)), m, n, lds)
        bad = _copy_check(A.data_ptr(), lds, m, n, M if copy else None, device) if (copy or check) else 0
    elif (isinstance(A, np.ndarray) and A.ndim == 2 and A.dtype == np.float64 and A.flags.c_contiguous
          and not A.flags.f_contiguous and A.nbytes >= _PIPELINE_MIN and not _is_pinned(A)):
        # C-ordered host input: pipelined upload of the rows, then the tiled
        # transpose + finite scan in one device pass (no host transpose)
        m, n = A.shape
        rows = torch.empty((m, n), dtype=torch.float64, device=device)
        _h2d_pipelined(A, rows)
        M = ColMajor.empty(m, n, device)
        cnt = torch.zeros(1, dtype=torch.int64, device=device)
        _lib.check(_lib.lib().sqr_copy_check_t(rows.data_ptr(), n, m, n, M.ptr, M.ld, cnt.data_ptr(),
                                               stream_handle()), "sqr_copy_check_t")
        bad = int(cnt.item()) if check else 0
    else:
        M = upload(A, device)
        bad = _copy_check(M.ptr, M.ld, M.m, M.n, None, device) if (check and M.m and M.n) else 0
    if bad:
        raise ValueError(f"A contains {bad} non-finite entries")
    return M


def check_finite(M: ColMajor, name: str = "A") -> None:
    if M.m and M.n:
        bad = _copy_check(M.ptr, M.ld, M.m, M.n, None, M.t.device)
        if bad:
            raise ValueError(f"{name} contains {bad} non-finite entries")


class Workspace:
    """Grow-only zero-initialised scratch, one per (device, CUDA stream).

    The reference promises "safe to call from multiple threads on disjoint
    data".  Calls on different streams therefore get
    different buffers (the cooperative kernels' grid-barrier words live in
    them), and calls sharing a stream hold that stream's lock for the whole
    enqueue (`lease`), so their kernels are stream-ordered one call after the
    other.  A grown buffer is allocated on its stream; the old one is
    released to torch's stream-ordered allocator when its last user drops
    it, never while a call that holds it is still enqueueing.  Barrier /
    semaphore words are left at zero by every kernel that uses them.
    """

    _cache: dict = {}
    _locks: dict = {}
    _guard = threading.Lock()

    @staticmethod
    def _key(device):
        dev = torch.device(device)
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        return (idx, torch.cuda.current_stream(idx).cuda_stream)

    @classmethod
    def _lock(cls, key) -> threading.RLock:
        with cls._guard:
            lk = cls._locks.get(key)
            if lk is None:
                lk = cls._locks[key] = threading.RLock()
            return lk

    @classmethod
    def get(cls, nbytes: int, device) -> torch.Tensor:
        """The current stream's buffer (>= nbytes).  Callers that enqueue
        several launches on it should hold `lease` instead."""
        key = cls._key(device)
        with cls._lock(key):
            buf = cls._cache.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.zeros(int(nbytes) + 4096, dtype=torch.uint8, device=torch.device("cuda", key[0]))
                cls._cache[key] = buf
            return buf

    @classmethod
    @contextlib.contextmanager
    def lease(cls, nbytes: int, device):
        """`with Workspace.lease(n, dev) as ws:` -- the buffer plus exclusive use
        of it (per stream) until the block has enqueued its kernels."""
        lk = cls._lock(cls._key(device))
        with lk:
            yield cls.get(nbytes, device)


def status_new(device) -> torch.Tensor:
    return torch.zeros(_lib.STATUS_BYTES, dtype=torch.uint8, device=device)


def status_read(st: torch.Tensor) -> np.void:
    host = st.cpu().numpy()
    return np.frombuffer(host.tobytes(), dtype=_lib.STATUS_DTYPE)[0]

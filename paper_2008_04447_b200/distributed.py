"""Multi-GPU RQRCP: 1-D column block-cyclic layout, one process per GPU
(north star: "column-partitioned block-cyclically across the
GPUs ... the replicated pivot decision on the small B is followed by an
NCCL-over-NVLink broadcast of the panel's Householder vectors and T, and each
GPU applies the trailing update to its own columns").

Global column block c (columns [c*b, (c+1)*b)) lives on rank c % P.  Per block
J of the reference loop (randomized.py:185-221):

  1. sample QRCP, replicated: every rank holds the identical sample B and runs
     the identical deterministic kernel, so pivots agree without messages;
  2. column moves: the <= 2b moved columns travel point to point (NCCL);
  3. panel: the owner of block J factors its local panel;
  4. broadcast of Y (m - i0 rows), taus, bhat and R11 from the owner;
  5. every rank applies the block reflection to its own trailing columns;
  6. every rank updates the sample for its own columns (sketch.py:132-149)
     and the slabs are all-gathered back into the replicated B.

The orchestration is written against two small interfaces -- ``comm``
(broadcast / all_gather / point-to-point, torch.distributed) and ``ops`` (the
local compute) -- so the same code runs on B200s (``GpuOps``: libsqr kernels,
NCCL) and, in the CPU test-suite, on gloo with a NumPy reference backend.
"""
from __future__ import annotations

import functools
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .counters import rqrcp_counters, trqrcp_counters

_DIAG_FLOOR = 2.0 ** -52


# ------------------------------------------------------------------ layout
@functools.lru_cache(maxsize=64)
def _local_columns(n: int, b: int, P: int, r: int) -> np.ndarray:
    nblk = -(-n // b)
    cols = [np.arange(c * b, min(n, (c + 1) * b), dtype=np.int64) for c in range(r, nblk, P)]
    out = np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)
    out.setflags(write=False)
    return out


@dataclass(frozen=True)
class BlockCyclic:
    """Column block-cyclic map with block width b over P ranks.  The per-rank
    column lists are computed once and cached (the driver asks for them every
    block)."""

    n: int
    b: int
    P: int

    @property
    def nblocks(self) -> int:
        return -(-self.n // self.b)

    def owner(self, p):
        return (np.asarray(p) // self.b) % self.P

    def local_index(self, p):
        p = np.asarray(p)
        c = p // self.b
        return (c // self.P) * self.b + p % self.b

    def blocks_of(self, r: int):
        return list(range(r, self.nblocks, self.P))

    def n_local(self, r: int) -> int:
        return int(_local_columns(self.n, self.b, self.P, r).size)

    def n_local_max(self) -> int:
        return self.n_local(0)  # rank 0 owns the first block, so never fewer columns

    def global_of_local(self, r: int) -> np.ndarray:
        """Global position of every local column of rank r, in local order
        (read-only cached array)."""
        return _local_columns(self.n, self.b, self.P, r)

    def first_local_at_or_after(self, r: int, p: int) -> int:
        """Local index of the first local column whose global position >= p."""
        return int(np.searchsorted(self.global_of_local(r), p))


@dataclass
class MovePlan:
    """Rank r's share of one block's column moves (dst <- src, global
    positions), in move order:
      pack      local indices of the sources this rank owns (read first);
      local     (packed row, local destination) pairs staying on this rank;
      send[q]   packed rows going to peer q;
      recv[q]   local destinations of the columns arriving from peer q.
    Every source is packed before any destination is written, so the moves
    act as one simultaneous permutation (randomized.py:194-195)."""

    pack: np.ndarray
    local_rows: np.ndarray
    local_dst: np.ndarray
    send: dict
    recv: dict


def move_plan(ps, pd, lay: BlockCyclic, r: int) -> MovePlan:
    ps, pd = np.asarray(ps), np.asarray(pd)
    osrc, odst = lay.owner(ps), lay.owner(pd)
    lsrc, ldst = lay.local_index(ps), lay.local_index(pd)
    mine = np.nonzero(osrc == r)[0]
    loc = np.nonzero(odst[mine] == r)[0]
    send = {int(q): np.nonzero(odst[mine] == q)[0] for q in sorted(set(odst[mine].tolist()) - {r})}
    recv = {}
    for q in sorted(set(osrc[odst == r].tolist()) - {r}):
        recv[int(q)] = ldst[np.nonzero((odst == r) & (osrc == q))[0]]
    return MovePlan(lsrc[mine], loc, ldst[mine[loc]], send, recv)


# -------------------------------------------------------------------- comm
class TorchComm:
    """torch.distributed with the process group's backend (NCCL on GPUs, gloo
    on CPU)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def broadcast(self, t: torch.Tensor, src: int) -> torch.Tensor:
        dist.broadcast(t, src=dist.get_global_rank(self.group, src) if self.group else src, group=self.group)
        return t

    def all_gather(self, t: torch.Tensor) -> list:
        outs = [torch.empty_like(t) for _ in range(self.size)]
        dist.all_gather(outs, t.contiguous(), group=self.group)
        return outs

    def exchange(self, sends: dict, recv_shapes: dict, like: torch.Tensor) -> dict:
        """Point-to-point: sends {peer: tensor}, receives {peer: tensor(shape)}."""
        ops, recvs = [], {}
        for peer, shape in sorted(recv_shapes.items()):
            buf = torch.empty(shape, dtype=like.dtype, device=like.device)
            recvs[peer] = buf
            ops.append(dist.P2POp(dist.irecv, buf, peer, group=self.group))
        for peer, t in sorted(sends.items()):
            ops.append(dist.P2POp(dist.isend, t.contiguous(), peer, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return recvs

    def max(self, x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64,
                         device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


def _gather_sample(ops, comm, slab, lay, p0, ell):
    """Replicated sample for positions >= p0 from every rank's slab: the ops'
    fused path if it has one (GpuOps over SymmComm: one put_columns kernel),
    else all-gather + assembly."""
    if hasattr(ops, "gather_sample"):
        return ops.gather_sample(slab, lay, p0, ell, comm)
    parts = comm.all_gather(ops.pad_slab(slab, lay, p0))
    return ops.assemble(parts, lay, ell) if p0 == 0 else ops.assemble_next(parts, lay, p0, ell)


class SymmComm(TorchComm):
    """TorchComm plus one symmetric device allocation for the device-initiated
    collectives of csrc/peer.cu (SURVEY.md §8(e) "B200-native upgrade"): the
    panel record and the replicated sample live in symmetric buffers, the
    producing rank's kernel stores into every peer's copy over NVLink and
    releases an epoch into the peers' flag words, consumers wait on the
    device.  No host-launched NCCL call and no host round trip sits between
    a producer and its consumers; the column moves keep NCCL point-to-point.

    Layout of the region: [flags: 2 kinds x P u64 | caller buffers ...];
    every rank holds the same layout, peer base pointers come from the
    torch.distributed._symmetric_memory rendezvous."""

    KIND_PANEL, KIND_SAMPLE = 0, 1

    def __init__(self, group=None, device=None):
        super().__init__(group)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.symm = True
        self.buf = None
        self.epochs = [0, 0]          # per kind; advanced identically on every rank
        self.counter = torch.zeros(16, dtype=torch.int32, device=self.dev)
        self.flag_bytes = ((2 * self.size * 8 + 255) // 256) * 256

    def allocate(self, nbytes: int) -> int:
        """Collective: (re)allocate the region with >= nbytes of caller space;
        returns the offset of the caller space."""
        import torch.distributed._symmetric_memory as symm_mem
        total = self.flag_bytes + int(nbytes)
        if self.buf is not None and self.buf.numel() >= total:
            return self.flag_bytes
        group = self.group if self.group is not None else dist.group.WORLD
        buf = symm_mem.empty(total, dtype=torch.uint8, device=self.dev)
        buf.zero_()
        self.h = symm_mem.rendezvous(buf, group.group_name)
        self.buf = buf
        self.base = [int(x) for x in self.h.buffer_ptrs]
        torch.cuda.synchronize(self.dev)
        self.h.barrier()
        self.epochs = [0, 0]
        return self.flag_bytes

    def peer_ptrs(self, offset: int, exclude_self: bool = False) -> torch.Tensor:
        ptrs = [b + offset for q, b in enumerate(self.base) if not (exclude_self and q == self.rank)]
        return torch.tensor(ptrs, dtype=torch.int64, device=self.dev)

    def flag_ptrs(self, exclude_self: bool = False) -> torch.Tensor:
        return self.peer_ptrs(0, exclude_self)

    def local_flags(self, kind: int) -> int:
        return self.buf.data_ptr() + 8 * kind * self.size

    def next_epoch(self, kind: int) -> int:
        self.epochs[kind] += 1
        return self.epochs[kind]


# ---------------------------------------------------------------- the loop
@dataclass
class DistResult:
    achieved: int
    nblocks: int
    reason: str
    perm: np.ndarray
    A_local: object          # this rank's columns: R rows / reflector tails packed (LAPACK style)
    taus: np.ndarray
    counters: object


def rqrcp_block_cyclic(A_local, m: int, n: int, k: int, b: int, p: int, seed: int, comm, ops,
                       omega=None) -> DistResult:
    """Distributed RQRCP (randomized.py:166-224) over ``comm``; ``A_local`` is
    this rank's block-cyclic column slab (ops-specific storage, m rows)."""
    ell = b + p
    lay = BlockCyclic(n, b, comm.size)
    r = comm.rank
    gloc = lay.global_of_local(r)
    if hasattr(ops, "begin"):
        ops.begin(lay, m, ell)
    perm = np.arange(n, dtype=np.int64)
    taus = np.zeros(max(k, 1))
    # 1. sketch: local slab, all-gathered into global column order.
    B = _gather_sample(ops, comm, ops.sketch(A_local, m, ell, seed, omega, gloc), lay, 0, ell)
    achieved, nblocks, reason = 0, 0, "k_reached"
    first = True
    # The panel's outcome (bhat, taus, R11) is read LAZILY: block J's trailing
    # update and sample update run assuming a complete panel (bhat = bb), and
    # its tail comes back with block J+1's sample-QRCP record in ONE host
    # synchronisation per block.  A short / zero panel or a singular R11 then
    # stops the loop exactly where the reference does (randomized.py:196-219):
    # the speculative work past that point is discarded, and the panel columns
    # left of a short panel's stop get the block update they miss.
    pend = None
    # Paired second sweep (as driver.cu's trailing_first / trailing_second,
    # randomized.py:203-210): with storage rows [m, m + 2b) per column (the
    # stacked W_P | W_J rows move with the column moves), block P = J - 1 of a
    # pair applies only its R12 rows and defers the rest of its update; J's
    # panel columns take P's update just before J's panel, J's first sweep is
    # corrected by (Y_J^T Y_P) W_P, and one K = 2b update applies both.
    pair_ok = (hasattr(ops, "block_update_defer") and A_local.shape[1] >= m + 2 * b
               and not os.environ.get("SQR_DIST_NO_PAIR"))
    pendP = None  # (i0, bb, pan, t0) of the block whose rows >= i0 + b still lack its update

    def flush():
        """Any exit while a block's update is deferred: apply the rest of it
        (the reference applied each block's full update before its next step)."""
        nonlocal pendP
        if pendP is not None:
            ops.flush_pending(A_local, pendP[3], pendP[0], m, pendP[2])
            pendP = None

    def settle(pd, tail, may_continue):
        """Apply the reference's exits for the pending block; True = stop."""
        nonlocal achieved, nblocks, reason
        pi0, pbb, pan, lc_owner = pd
        bhat, taus_host, r11_diag = tail
        if bhat == 0:  # randomized.py:197: no block, no update (ours used Y = 0: a no-op)
            achieved, nblocks, reason = pi0, nblocks - 1, "panel_zero"
            return True
        taus[pi0:pi0 + bhat] = taus_host[:bhat]
        if bhat < pbb:
            # the short panel's remaining columns also take the block update
            if lc_owner >= 0:
                ops.block_update(A_local, lc_owner + bhat, pi0, m, pan, ncols=pbb - bhat)
            achieved, reason = pi0 + bhat, "short_block"
            return True
        if not may_continue:
            return True
        d = np.abs(r11_diag)
        if not (d.size > 0 and d.min() > _DIAG_FLOOR * d[0]):
            reason = "r11_singular"
            return True
        return False

    while achieved < k:
        i0 = achieved
        bb = min(b, k - i0)
        nt = n - i0
        # ---- replicated sample QRCP (identical input -> identical pivots)
        samp = ops.sample_qrcp(B, ell, nt, bb, first, pend[2] if pend else None)
        first = False
        if pend is not None:
            stop = settle(pend, samp.prev_tail, True)
            pend = None
            if stop:
                flush()
                break
        if samp.stop:
            reason = samp.reason
            flush()
            break
        # ---- column moves (positions relative to i0)
        moves = samp.moves
        if len(moves):
            ps = i0 + moves[:, 1]
            pd = i0 + moves[:, 0]
            ops.move_columns(A_local, ps, pd, lay, comm, i0=i0, samp=samp)
            perm[pd] = perm[ps].copy()
        # ---- panel on the owner, broadcast of (Y, taus, bhat, R11)
        J = i0 // b
        owner = J % comm.size
        lc = int(lay.local_index(i0)) if owner == r else -1
        if pendP is not None and owner == r:  # J's panel columns get the deferred P first
            ops.pending_panel(A_local, lc, i0, m, samp.achieved, pendP)
        pan = ops.panel(A_local, lc, i0, m, samp.achieved, bb, owner == r)
        pan = ops.broadcast_panel(pan, owner, comm, m - i0, bb)
        if hasattr(ops, "prep_sample_update"):  # overlaps the trailing update
            ops.prep_sample_update(samp, pan, bb)
        # ---- trailing update of my columns at global positions >= i0 + bb
        t0 = lay.first_local_at_or_after(r, i0 + bb)
        last = i0 + bb >= k or n - (i0 + bb) == 0
        if pendP is not None:
            ops.block_update_merge(A_local, t0, i0, m, pan, pendP)
            pendP = None
        elif pair_ok and not last and bb == b and i0 + 2 * b <= k:
            ops.block_update_defer(A_local, t0, i0, m, pan)
            pendP = (i0, bb, pan, t0)
        else:
            ops.block_update(A_local, t0, i0, m, pan)
        nblocks += 1
        achieved = i0 + bb
        pend = (i0, bb, pan, lc)
        if achieved >= k:
            reason = "k_reached"
            break
        if n - achieved == 0:
            reason = "no_trailing"
            break
        # ---- sample update for my columns, all-gathered (sketch.py:132-149)
        s0 = lay.first_local_at_or_after(r, achieved)
        mine = gloc[s0:]
        Bn_loc = ops.sample_update_local(samp, A_local, s0, mine - i0, i0, bb, pan)
        B = _gather_sample(ops, comm, Bn_loc, lay, achieved, ell)
    if pend is not None:
        settle(pend, ops.read_tail(pend[2]), False)
    flush()
    if hasattr(ops, "finish"):
        ops.finish()
    counters = rqrcp_counters(m, n, b, ell, achieved, nblocks,
                              {"k_reached": 1, "short_block": 5, "no_trailing": 6}.get(reason, 0), False)
    return DistResult(achieved, nblocks, reason, perm, A_local, taus[:achieved], counters)


def trqrcp_block_cyclic(S_local, m: int, n: int, k: int, b: int, p: int, seed: int, comm, ops,
                        omega=None) -> DistResult:
    """Distributed TRQRCP (randomized.py:250-341), same column block-cyclic
    layout.  ``S_local`` stacks, per local column, the reference's three
    column-permuted arrays: rows [0, m) = work (A, never updated), [m, m+k) =
    Wg (W^T rows), [m+k, m+2k) = Rg (R rows) -- so one column move carries all
    three (randomized.py:299-302).  Yg (m x k) is replicated: every rank
    stores the broadcast panel reflectors.  Per block: replicated sample QRCP;
    column moves; the owner materialises its panel through the accumulated
    reflections and factors it (:304-307); broadcast of (Y, taus, R11); every
    rank forms the adjusted inner products, W^T rows and R rows of its OWN
    trailing columns (:318-330, all column-local); local sample update +
    all-gather.  The panel tail is read synchronously (TRQRCP runs few blocks).
    Returns a DistResult with A_local = S_local and ``Yg``/``nb`` attached."""
    ell = b + p
    lay = BlockCyclic(n, b, comm.size)
    r = comm.rank
    gloc = lay.global_of_local(r)
    if hasattr(ops, "begin"):
        ops.begin(lay, m, ell)
    perm = np.arange(n, dtype=np.int64)
    taus = np.zeros(max(k, 1))
    B = _gather_sample(ops, comm, ops.sketch(S_local, m, ell, seed, omega, gloc), lay, 0, ell)
    Yg = ops.new_yg(m, k)
    achieved, nblocks, reason = 0, 0, "k_reached"
    first = True
    while achieved < k:
        i0 = achieved
        bb = min(b, k - i0)
        nt = n - i0
        samp = ops.sample_qrcp(B, ell, nt, bb, first)
        first = False
        if samp.stop:
            reason = samp.reason
            break
        moves = samp.moves
        if len(moves):
            ps = i0 + moves[:, 1]
            pd = i0 + moves[:, 0]
            ops.move_columns(S_local, ps, pd, lay, comm)
            perm[pd] = perm[ps].copy()
        owner = (i0 // b) % comm.size
        lc = int(lay.local_index(i0)) if owner == r else -1
        pan = ops.tr_panel(S_local, lc, i0, m, k, samp.achieved, bb, owner == r, Yg)
        pan = ops.broadcast_panel(pan, owner, comm, m - i0, bb)
        bhat, taus_h, r11_diag = ops.read_tail(pan)
        if bhat == 0:                                   # randomized.py:308-309
            reason = "panel_zero"
            break
        taus[i0:i0 + bhat] = taus_h[:bhat]
        nblocks += 1
        t0 = lay.first_local_at_or_after(r, i0 + bhat)
        ops.tr_update(S_local, t0, i0, m, k, pan, bhat, Yg, lc)
        achieved = i0 + bhat
        if bhat < bb:                                   # randomized.py:332-333
            reason = "short_block"
            break
        if achieved >= k:
            reason = "k_reached"
            break
        if n - achieved == 0:
            reason = "no_trailing"
            break
        d = np.abs(r11_diag)
        if not (d.size > 0 and d.min() > _DIAG_FLOOR * d[0]):   # randomized.py:334-335
            reason = "r11_singular"
            break
        s0 = lay.first_local_at_or_after(r, achieved)
        mine = gloc[s0:]
        Bn_loc = ops.sample_update_local(samp, S_local, s0, mine - i0, i0, bb, pan, r_row0=m + k + i0)
        B = _gather_sample(ops, comm, Bn_loc, lay, achieved, ell)
    counters = trqrcp_counters(m, n, b, ell, achieved, nblocks)
    res = DistResult(achieved, nblocks, reason, perm, S_local, taus[:achieved], counters)
    res.Yg = Yg
    return res


# ------------------------------------------------------------ GPU backend
@dataclass
class _Sample:
    stop: bool
    reason: str
    achieved: int
    moves: np.ndarray
    Bf: object
    st: object
    prev_tail: object = None  # (bhat, taus, diag R11) of the previous block's panel, read with this record


@dataclass
class _Panel:
    bhat: int
    Y: object            # (bb, mr) column-major explicit unit-lower Y
    taus: object         # device (bb,)
    taus_host: np.ndarray
    R11: object          # (bb, bb) device
    R11_host: np.ndarray
    st: object
    tail: object = None  # device [taus | R11 | status] record, parsed lazily


class GpuOps:
    """libsqr kernels on torch CUDA tensors; matrices are (ncols, ld) tensors.

    Every per-block buffer is allocated once per factorization shape and
    reused; per block the host reads back two small control records (the
    sample QRCP status + moves, and the broadcast panel tail: status, taus,
    R11) and uploads one packed index array for the column moves."""

    def __init__(self, device, comm=None):
        from . import _lib
        from ._dev import Workspace
        self.L = _lib.lib()
        self.lib = _lib
        self.dev = torch.device(device)
        self.Workspace = Workspace
        self._keep = []
        self._shape = None
        self._stage_h = self._stage_np = self._stage_d = None
        self._stage_used = 0
        self._tail = None       # deferred rows of a merged second sweep (lookahead)
        self._stream = torch.cuda.current_stream(self.dev)
        self._sh = self._stream.cuda_stream
        self.lookahead = not os.environ.get("SQR_DIST_NO_LOOKAHEAD")
        # the deferred rows run BESIDE the next sample QRCP (a whole-SM kernel on ceil(n_t / 256) SMs)
        # on their own stream, released once that kernel is resident (csrc/driver.cu Overlap)
        self.beside = self.lookahead and not os.environ.get("SQR_DIST_NO_BESIDE")
        self.plan_moves = bool(os.environ.get("SQR_DIST_PLAN_MOVES"))   # world 1: exercise the P2P plan path
        # SymmComm: panel broadcast and sample all-gather as device-initiated
        # NVLink puts into symmetric buffers (csrc/peer.cu)
        self.symm = comm if getattr(comm, "symm", False) else None

    # helpers
    def _s(self):
        return self._sh   # the caller's current stream, fixed per factorization (begin)

    def _cur(self):
        return self._stream

    def _ws(self, nbytes):
        return self.Workspace.get(nbytes, self.dev)

    def _chk(self, rc, what):
        self.lib.check(rc, what)

    def _idx(self, a):
        """Upload an index list (asynchronously).  Bump-allocated from one
        pinned staging buffer and its device twin, both reset at the per-block
        host synchronisation: every copy and kernel enqueued before it has
        finished by then (stream order), so neither side is reused early."""
        a = np.asarray(a, dtype=np.int64)
        n = a.size
        if self._stage_h is not None and self._stage_used + n <= self._stage_h.numel():
            o = self._stage_used
            self._stage_used = o + ((n + 15) // 16) * 16
            self._stage_np[o:o + n] = a
            d = self._stage_d[o:o + n]
            d.copy_(self._stage_h[o:o + n], non_blocking=True)
            return d
        # overflow (never at the shapes the driver uses): a private pinned copy,
        # kept alive until the next sync point
        t = torch.as_tensor(a).pin_memory().to(self.dev, non_blocking=True)
        self._keep.append(t)
        return t

    def _synced(self):
        self._stage_used = 0
        self._keep.clear()

    def begin(self, lay, m, ell):
        """Per-shape persistent buffers (allocated on the first call of a
        factorization of this shape)."""
        self._stream = torch.cuda.current_stream(self.dev)
        self._sh = self._stream.cuda_stream
        self._P = lay.P
        key = (lay.n, lay.b, lay.P, m, ell)
        if self._shape == key:
            return
        self._shape = key
        n, b = lay.n, lay.b
        self.b = b
        f64 = dict(dtype=torch.float64, device=self.dev)
        prec = ((b * m + b + b * b + 9) + 1) // 2 * 2                  # panel record doubles (16-byte multiple)
        if self.symm is not None:
            # double-buffered (block parity) panel records and replicated samples
            bg = max(n, 1) * ell
            off = self.symm.allocate(8 * 2 * (bg + prec))
            base = self.symm.buf[off:off + 8 * 2 * (bg + prec)].view(torch.float64)
            self.Bglobs = [base[i * bg:(i + 1) * bg].view(max(n, 1), ell) for i in range(2)]
            self.pbufs = [base[2 * bg + i * prec:2 * bg + (i + 1) * prec] for i in range(2)]
            self.off_B = [off + 8 * i * bg for i in range(2)]
            self.off_P = [off + 8 * (2 * bg + i * prec) for i in range(2)]
            self.put_B = [self.symm.peer_ptrs(o) for o in self.off_B]
            self.put_P = [self.symm.peer_ptrs(o, exclude_self=True) for o in self.off_P]
            self.flags_all = self.symm.flag_ptrs()
            self.flags_peers = self.symm.flag_ptrs(exclude_self=True)
            self.Bglob = self.Bglobs[0]
            self.pbuf = self.pbufs[0]
        else:
            self.Bglob = torch.zeros((max(n, 1), ell), **f64)            # replicated sample, global positions
        self.Bf = torch.zeros((max(n, 1), ell), **f64)
        self.lperm = torch.zeros(max(n, 1), dtype=torch.int64, device=self.dev)
        self.ctl = torch.zeros(128 + 4 * (4 * b + 8), dtype=torch.uint8, device=self.dev)
        self.staus = torch.zeros(b, **f64)
        # panel broadcast record: [Y (b x m) | taus (b) | R11 (b x b) | status (9 doubles)]
        if self.symm is None:
            self.pbufs = [torch.zeros(prec, **f64) for _ in range(2)]
            self.pbuf = self.pbufs[0]
        self.T = torch.zeros((b, b), **f64)
        nmax = lay.n_local_max()
        self.slab = torch.zeros((max(nmax, 1), ell), **f64)
        self.Bfl = torch.zeros((b + max(nmax, 1), ell), **f64)
        self.Rl = torch.zeros((b + max(nmax, 1), b), **f64)
        self.mbuf = torch.zeros(b * b, **f64)
        self.sws = torch.zeros(int(self.L.sqr_sample_qrcp_workspace(ell, n)), dtype=torch.uint8, device=self.dev)
        self.side = torch.cuda.Stream(self.dev, priority=-1)
        self.bulk = torch.cuda.Stream(self.dev)
        self.sig = torch.zeros(16, dtype=torch.int32, device=self.dev)
        self._epoch = 0
        self.prep_done = None
        self.h_ctl = torch.zeros(self.ctl.numel(), dtype=torch.uint8).pin_memory()
        self.h_ctl_i32 = self.h_ctl.numpy().view(np.int32)
        self.h_ctl_f64 = self.h_ctl.numpy()[:72].view(np.float64)
        self.h_tail = torch.zeros(b + b * b + 9, dtype=torch.float64).pin_memory()
        self.h_tail_np = self.h_tail.numpy()
        self.gidx = [torch.tensor(lay.global_of_local(q), device=self.dev) for q in range(lay.P)]
        ns = 2 * max(nmax, 1) + 64 * b + 1024
        self._stage_h = torch.zeros(ns, dtype=torch.int64).pin_memory()
        self._stage_np = self._stage_h.numpy()
        self._stage_d = torch.zeros(ns, dtype=torch.int64, device=self.dev)
        self._stage_used = 0

    # 1. sketch of the local slab
    def sketch(self, A, m, ell, seed, omega, gloc):
        OmT = torch.empty((ell, m), dtype=torch.float64, device=self.dev)  # Omega^T: m x ell column-major
        if omega is None:
            self._chk(self.L.sqr_gaussian(OmT.data_ptr(), m, ell, m, seed & ((1 << 64) - 1), 0, 1, self._s()),
                      "sqr_gaussian")
        else:
            OmT.copy_(torch.as_tensor(np.ascontiguousarray(np.asarray(omega, dtype=np.float64)), device=self.dev))
        nl = A.shape[0]
        Bl = torch.empty((max(nl, 1), ell), dtype=torch.float64, device=self.dev)
        if nl:
            ws = self._ws(200 << 20)
            self._chk(self.L.sqr_gemm_tn(ell, nl, m, 1.0, OmT.data_ptr(), m, A.data_ptr(), A.shape[1], 0.0, None, 0,
                                         Bl.data_ptr(), ell, ws.data_ptr(), ws.numel(), self._s()), "sketch")
        return Bl

    def pad_slab(self, Bn, lay, achieved):
        if Bn.data_ptr() == self.slab.data_ptr():
            return self.slab          # the sample update wrote straight into the slab
        nb = min(Bn.shape[0], self.slab.shape[0])
        if nb:
            self.slab[:nb].copy_(Bn[:nb])
        return self.slab

    def _assemble(self, parts, lay, ell, p0):
        """Columns of the all-gathered slabs into the replicated sample at their
        global positions; the sample for positions >= p0 is Bglob[p0:]."""
        for q, part in enumerate(parts):
            s = lay.first_local_at_or_after(q, p0)
            cnt = lay.n_local(q) - s
            if cnt > 0:
                self._chk(self.L.sqr_copy_columns(part.data_ptr(), ell, ell, None, self.Bglob.data_ptr(), ell,
                                                  self.gidx[q][s:].data_ptr(), cnt, self._s()), "assemble")
        return self.Bglob[p0:]

    def assemble(self, parts, lay, ell):
        return self._assemble(parts, lay, ell, 0)

    def gather_sample(self, slab, lay, p0, ell, comm):
        """Replicated sample for positions >= p0.  SymmComm: this rank's slab
        columns go straight to their global positions in every peer's sample
        (one sqr_peer_put_columns: all-gather + assembly), then a device-side
        wait for every rank's epoch.  Else NCCL all-gather + assembly."""
        if self.symm is None:
            if comm.size == 1 and slab.data_ptr() == self.Bglob[p0:].data_ptr():
                return self.Bglob[p0:]     # already in place (sample_update_local)
            parts = comm.all_gather(self.pad_slab(slab, lay, p0))
            return self._assemble(parts, lay, ell, p0)
        sy = self.symm
        par = (p0 // lay.b) & 1
        ep = sy.next_epoch(sy.KIND_SAMPLE)
        s0 = lay.first_local_at_or_after(comm.rank, p0)
        cnt = lay.n_local(comm.rank) - s0
        self._chk(self.L.sqr_peer_put_columns(slab.data_ptr(), ell, ell, max(cnt, 0),
                                              self.gidx[comm.rank][s0:].data_ptr(), self.put_B[par].data_ptr(), ell,
                                              comm.size, self.flags_all.data_ptr(), sy.KIND_SAMPLE * comm.size
                                              + comm.rank, ep, sy.counter.data_ptr(), self._s()), "peer_put_columns")
        self._chk(self.L.sqr_peer_wait(sy.local_flags(sy.KIND_SAMPLE), comm.size, ep, self._s()), "peer_wait")
        self.Bglob = self.Bglobs[par]
        return self.Bglob[p0:]

    def _select_panel_buffer(self, i0):
        # by block parity: a deferred block P's record (Y_P) must survive J's panel
        self.pbuf = self.pbufs[(i0 // self.b) & 1]

    def assemble_next(self, parts, lay, achieved, ell):
        return self._assemble(parts, lay, ell, achieved)

    # 2. replicated sample QRCP
    def _join_prep(self):
        if self.prep_done is not None:
            self._cur().wait_event(self.prep_done)
            self.prep_done = None

    def sample_qrcp(self, B, ell, nt, bb, first, pend_pan=None):
        self._join_prep()  # the overlapped prep writes the status record zeroed below
        st = self.ctl[:72]
        st.zero_()
        if not first:  # the sample floor of the first block (randomized.py:179-180)
            st[32:40].view(torch.float64).fill_(self._floor)
        moves = self.ctl[128:].view(torch.int32)
        beside = self.beside and self._tail is not None
        if beside:
            # deferred rows of the merged second sweep beside this kernel (see __init__)
            self._epoch += 1
            ready = torch.cuda.Event()
            ready.record(self._cur())
            self._chk(self.L.sqr_sample_qrcp_ws_sig(B.data_ptr(), ell, ell, nt, bb, self.Bf.data_ptr(), ell,
                                                    self.lperm.data_ptr(), moves.data_ptr(), self.staus.data_ptr(),
                                                    1 if first else 0, st.data_ptr(), self.sws.data_ptr(),
                                                    self.sws.numel(), self.sig.data_ptr(), self._epoch, self._s()),
                      "sample_qrcp")
            self.bulk.wait_event(ready)
            self._chk(self.L.sqr_wait_resident(self.sig.data_ptr(), self._epoch, 100, self.bulk.cuda_stream),
                      "wait_resident")
            self.run_tail(self.bulk.cuda_stream)
            bulk_done = torch.cuda.Event()
            bulk_done.record(self.bulk)
        else:
            self._chk(self.L.sqr_sample_qrcp_ws(B.data_ptr(), ell, ell, nt, bb, self.Bf.data_ptr(), ell,
                                                self.lperm.data_ptr(), moves.data_ptr(), self.staus.data_ptr(),
                                                1 if first else 0, st.data_ptr(), self.sws.data_ptr(),
                                                self.sws.numel(), self._s()), "sample_qrcp")
        # one host synchronisation: status + moves, plus the previous panel's tail;
        # without `beside` the deferred rows of a merged second sweep run behind it (lookahead)
        self.h_ctl.copy_(self.ctl, non_blocking=True)
        if pend_pan is not None:
            self.h_tail[:pend_pan.tail.numel()].copy_(pend_pan.tail, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(self._cur())
        if beside:
            self._cur().wait_event(bulk_done)   # the column moves that follow touch the same rows
        else:
            self.run_tail()
        ev.synchronize()
        self._synced()
        prev_tail = self._parse_tail(self.h_tail_np, pend_pan.Y.shape[0]) if pend_pan is not None else None
        hi = self.h_ctl_i32       # sqr_status words: stop, reason, .., sample_achieved (4), .., nmoves (6)
        if first:
            self._floor = float(self.h_ctl_f64[4])   # floor_sq (byte 32)
        stop = bool(hi[0])
        reason = {2: "sample_floor", 3: "sample_rank"}.get(int(hi[1]), "none")
        nm = int(hi[6])
        mv = hi[32:32 + 2 * nm].reshape(nm, 2).astype(np.int64)   # moves (byte 128): (dst, src) pairs
        mv = mv[(mv[:, 0] >= 0) & (mv[:, 0] != mv[:, 1])]  # drop no-op slots (dst = -1) and self-moves
        smp = _Sample(stop, reason, int(hi[4]), mv, self.Bf[:max(nt, 1)], st)
        smp.prev_tail = prev_tail
        return smp

    # 3. point-to-point column moves
    def move_columns(self, A, ps, pd, lay, comm, i0=None, samp=None):
        ld = A.shape[1]
        if comm.size == 1 and samp is not None and not self.plan_moves:
            # a world of one: every move is local -- the sample QRCP's device
            # move list drives the register-staged permutation kernel directly
            # (the single-GPU driver's apply_moves), no host plan or packing
            nmv = 2 * self.b
            self._chk(self.L.sqr_apply_moves(A.data_ptr(), ld, ld, i0, None, self.ctl[128:].data_ptr(),
                                             samp.st.data_ptr(), nmv, self._s()), "apply_moves")
            return
        plan = move_plan(ps, pd, lay, comm.rank)
        peers_out, peers_in = list(plan.send), list(plan.recv)
        # one upload for every index list of this block
        pieces = ([plan.pack, plan.local_rows, plan.local_dst] + [plan.send[q] for q in peers_out]
                  + [plan.recv[q] for q in peers_in])
        offs = np.cumsum([0] + [p.size for p in pieces])
        dev_idx = self._idx(np.concatenate(pieces) if offs[-1] else np.zeros(1, np.int64))

        def view(i):
            return dev_idx[offs[i]:offs[i + 1]]

        sends, recv_shapes = {}, {}
        packed = None
        if plan.pack.size:
            packed = torch.empty((plan.pack.size, ld), dtype=torch.float64, device=self.dev)
            self._chk(self.L.sqr_copy_columns(A.data_ptr(), ld, ld, view(0).data_ptr(), packed.data_ptr(), ld, None,
                                              plan.pack.size, self._s()), "pack")
            for i, q in enumerate(peers_out):
                sends[q] = packed.index_select(0, view(3 + i))
        for q in peers_in:
            recv_shapes[q] = (int(plan.recv[q].size), ld)
        recvs = comm.exchange(sends, recv_shapes, A)
        # unpack: local moves then received columns, in move order per source
        if plan.local_rows.size:
            self._chk(self.L.sqr_copy_columns(packed.data_ptr(), ld, ld, view(1).data_ptr(), A.data_ptr(), ld,
                                              view(2).data_ptr(), plan.local_rows.size, self._s()), "unpack")
        for i, q in enumerate(peers_in):
            buf = recvs[q]
            self._chk(self.L.sqr_copy_columns(buf.data_ptr(), ld, ld, None, A.data_ptr(), ld,
                                              view(3 + len(peers_out) + i).data_ptr(), buf.shape[0], self._s()),
                      "unpack")

    # 4. panel on the owner + broadcast
    def _panel_views(self, mr, bb):
        y = bb * mr
        Y = self.pbuf[:y].view(bb, mr)
        taus = self.pbuf[y:y + bb]
        R11 = self.pbuf[y + bb:y + bb + bb * bb].view(bb, bb)
        st = self.pbuf[y + bb + bb * bb:y + bb + bb * bb + 9].view(torch.uint8)
        return Y, taus, R11, st, self.pbuf[:y + bb + bb * bb + 9], self.pbuf[y:y + bb + bb * bb + 9]

    def panel(self, A, lc, i0, m, w, bb, is_owner):
        self._select_panel_buffer(i0)
        mr = m - i0
        Y, taus, R11, st, rec, tail = self._panel_views(mr, bb)
        if is_owner:
            rec.zero_()
            ld = A.shape[1]
            Pp = A.data_ptr() + 8 * (lc * ld + i0)
            ws = self._ws(self.L.sqr_block_workspace(mr, 0, bb))
            self._chk(self.L.sqr_panel_factor(Pp, ld, mr, w, Y.data_ptr(), mr, taus.data_ptr(), 1, st.data_ptr(),
                                              ws.data_ptr(), ws.numel(), self._s()), "panel")
            R11.copy_(A[lc:lc + bb, i0:i0 + bb])
        return _Panel(0, Y, taus, None, R11, None, st)

    def broadcast_panel(self, pan, owner, comm, mr, bb):
        _, _, _, _, rec, tail = self._panel_views(mr, bb)
        if self.symm is None:
            comm.broadcast(rec, owner)       # one message: Y, taus, R11, status
        elif comm.size > 1:
            # the owner stores the record into every peer's copy (NVLink P2P)
            # and releases the epoch; the others gate their stream on it
            sy = self.symm
            ep = sy.next_epoch(sy.KIND_PANEL)
            par = 0 if self.pbuf.data_ptr() == self.pbufs[0].data_ptr() else 1
            if comm.rank == owner:
                nbytes = ((rec.numel() * 8 + 15) // 16) * 16
                self._chk(self.L.sqr_peer_put(rec.data_ptr(), nbytes, self.put_P[par].data_ptr(), 0, comm.size - 1,
                                              self.flags_peers.data_ptr(), sy.KIND_PANEL * comm.size + owner, ep,
                                              sy.counter.data_ptr() + 4, self._s()), "peer_put")
            else:
                self._chk(self.L.sqr_peer_wait(sy.local_flags(sy.KIND_PANEL) + 8 * owner, 1, ep, self._s()),
                          "peer_wait")
        pan.tail = tail                      # read with the next block's sample record
        return pan

    @staticmethod
    def _parse_tail(h, bb):
        """(bhat, taus, diag R11[:bhat]) from a [taus | R11 | status] record
        (the drivers read only R11's diagonal: randomized.py:217-219, 334-335)."""
        meta = h[bb + bb * bb:bb + bb * bb + 9].view(np.int32)
        bhat = 0 if meta[0] else int(meta[5])
        d = h[bb:bb + bb * bb:bb + 1][:bhat].copy()   # (bb, bb) column-major: stride bb + 1
        return bhat, h[:bb].copy(), d

    def read_tail(self, pan):
        self._join_prep()
        self.run_tail()
        out = self._parse_tail(pan.tail.cpu().numpy(), pan.Y.shape[0])
        self._synced()
        return out

    def run_tail(self, stream=None):
        """Enqueue the deferred rows >= i0 + bb of the last merged second sweep."""
        if self._tail is not None:
            M, N, K, X, ldx, W, ld, C = self._tail
            self._tail = None
            if stream is None:
                self._gemm_nn(M, N, K, 1.0, X, ldx, W, ld, 1.0, C, ld, C, ld)
            elif M > 0 and N > 0:
                self._chk(self.L.sqr_gemm_nn(M, N, K, 1.0, X, ldx, W, ld, 1.0, C, ld, C, ld, stream), "gemm_nn")

    def finish(self):
        self.run_tail()

    # 4b. sample-update prep (R11 guard, M = S11 R11^-1) on a high-priority side
    #     stream while the trailing update runs (cf. driver.cu EarlyPrep)
    def prep_sample_update(self, samp, pan, bb):
        ev = torch.cuda.Event()
        ev.record(self._cur())
        self.side.wait_event(ev)
        ell = samp.Bf.shape[1]
        self._chk(self.L.sqr_sample_update_prep(samp.Bf.data_ptr(), ell, pan.R11.data_ptr(), bb, bb,
                                                self.mbuf.data_ptr(), samp.st.data_ptr(), self.side.cuda_stream),
                  "sample_update_prep")
        self.prep_done = torch.cuda.Event()
        self.prep_done.record(self.side)

    # 5. trailing update of my columns
    def block_update(self, A, t0, i0, m, pan, ncols=None):
        ld = A.shape[1]
        ncols = A.shape[0] - t0 if ncols is None else ncols
        bb = pan.Y.shape[0]
        mr = m - i0
        T = self.T.view(-1)[:bb * bb].view(bb, bb)
        ws = self._ws(self.L.sqr_block_workspace(mr, max(ncols, 0), bb))
        self._chk(self.L.sqr_apply_block_update(A.data_ptr() + 8 * (t0 * ld + i0), ld, mr, max(ncols, 0), bb,
                                                pan.Y.data_ptr(), mr, pan.taus.data_ptr(), T.data_ptr(), bb,
                                                ws.data_ptr(), ws.numel(), self._s()), "block_update")
        pan.T = T

    # 5b. paired second sweep (storage rows [m, m + b) = W_P, [m + b, m + 2b) = W_J)
    def _build_t(self, Y, mr, bb, taus):
        T = torch.empty((bb, bb), dtype=torch.float64, device=self.dev)
        ws = self._ws(200 << 20)
        self._chk(self.L.sqr_build_t(Y.data_ptr(), mr, mr, bb, taus.data_ptr(), T.data_ptr(), bb, ws.data_ptr(),
                                     ws.numel(), self._s()), "build_t")
        return T

    def _scratch(self, name, numel):
        buf = getattr(self, name, None)
        if buf is None or buf.numel() < numel:
            buf = torch.empty(max(numel, 1), dtype=torch.float64, device=self.dev)
            setattr(self, name, buf)
        return buf

    def block_update_defer(self, A, t0, i0, m, pan):
        """Block P of a pair: W_P = -T^T Y^T C into the W_P rows, and only the R12
        rows C[i0:i0+b] += Y[:b] W_P (the sample update needs them)."""
        ld = A.shape[1]
        bb, mr = pan.Y.shape[0], m - i0
        ncols = A.shape[0] - t0
        T = self._build_t(pan.Y, mr, bb, pan.taus)
        pan.T = T
        if ncols <= 0:
            return
        base = A.data_ptr() + 8 * t0 * ld
        C, Wp = base + 8 * i0, base + 8 * m
        Wt = self._scratch("_wt", bb * ncols)
        self._gemm_tn(bb, ncols, mr, 1.0, pan.Y.data_ptr(), mr, C, ld, Wt.data_ptr(), bb)
        self._gemm_tn(bb, ncols, bb, -1.0, T.data_ptr(), bb, Wt.data_ptr(), bb, Wp, ld)
        self._gemm_nn(bb, ncols, bb, 1.0, pan.Y.data_ptr(), mr, Wp, ld, 1.0, C, ld, C, ld)

    def pending_panel(self, A, lc, i0, m, w, pendP):
        """J's panel columns (owner) take the deferred P on rows >= i0, then
        their W_P is retired (a short panel never sees P twice)."""
        pi0, b, ppan, _ = pendP
        ld, mrP = A.shape[1], m - pi0
        if w <= 0:
            return
        col = A.data_ptr() + 8 * lc * ld
        self._gemm_nn(m - i0, w, b, 1.0, ppan.Y.data_ptr() + 8 * (i0 - pi0), mrP, col + 8 * m, ld, 1.0,
                      col + 8 * i0, ld, col + 8 * i0, ld)
        A[lc:lc + w, m:m + b].zero_()

    def block_update_merge(self, A, t0, i0, m, pan, pendP):
        """Block J of a pair: [Y_J^T C] + (Y_J^T Y_P) W_P (C still lacks P),
        W_J = -T_J^T (.), then C += [Y_P | Y_J] [W_P ; W_J] with K = b + bb."""
        pi0, b, ppan, _ = pendP
        ld = A.shape[1]
        bb, mr, mrP = pan.Y.shape[0], m - i0, m - pi0
        ncols = A.shape[0] - t0
        T = self._build_t(pan.Y, mr, bb, pan.taus)
        pan.T = T
        if ncols <= 0:
            return
        base = A.data_ptr() + 8 * t0 * ld
        C, Wp, Wj = base + 8 * i0, base + 8 * m, base + 8 * (m + b)
        Ypj = ppan.Y.data_ptr() + 8 * (i0 - pi0)          # Y_P rows from i0, ld mrP
        Wt = self._scratch("_wt", bb * ncols)
        X = self._scratch("_yjyp", bb * b)
        self._gemm_tn(bb, ncols, mr, 1.0, pan.Y.data_ptr(), mr, C, ld, Wt.data_ptr(), bb)
        self._gemm_tn(bb, b, mr, 1.0, pan.Y.data_ptr(), mr, Ypj, mrP, X.data_ptr(), bb)
        self._gemm_nn(bb, ncols, b, 1.0, X.data_ptr(), bb, Wp, ld, 1.0, Wt.data_ptr(), bb, Wt.data_ptr(), bb)
        self._gemm_tn(bb, ncols, bb, -1.0, T.data_ptr(), bb, Wt.data_ptr(), bb, Wj, ld)
        Ycat = self._scratch("_ycat", (b + bb) * mr)[:(b + bb) * mr].view(b + bb, mr)
        Ycat[:b].copy_(ppan.Y[:, i0 - pi0:])
        Ycat[b:].copy_(pan.Y)
        if self.lookahead and mr > bb:
            # the R12 rows now (the sample update reads them); the rows below
            # run after the next block's sample QRCP is launched, so they cover
            # that block's host synchronisation (run_tail)
            self._gemm_nn(bb, ncols, b + bb, 1.0, Ycat.data_ptr(), mr, Wp, ld, 1.0, C, ld, C, ld)
            self._tail = (mr - bb, ncols, b + bb, Ycat.data_ptr() + 8 * bb, mr, Wp, ld, C + 8 * bb)
        else:
            self._gemm_nn(mr, ncols, b + bb, 1.0, Ycat.data_ptr(), mr, Wp, ld, 1.0, C, ld, C, ld)

    def flush_pending(self, A, t0, i0, m, pan):
        """The deferred rows >= i0 + b of a block whose pair partner never came."""
        ld, b, mr = A.shape[1], pan.Y.shape[0], m - i0
        ncols = A.shape[0] - t0
        if ncols <= 0 or mr <= b:
            return
        base = A.data_ptr() + 8 * t0 * ld
        self._gemm_nn(mr - b, ncols, b, 1.0, pan.Y.data_ptr() + 8 * b, mr, base + 8 * m, ld, 1.0,
                      base + 8 * (i0 + b), ld, base + 8 * (i0 + b), ld)

    # TRQRCP (trqrcp_block_cyclic): replicated Yg, panel materialisation, local W^T / R rows
    def new_yg(self, m, k):
        return torch.zeros((max(k, 1), m), dtype=torch.float64, device=self.dev)   # m x k column-major

    def _gemm_tn(self, M, N, K, alpha, X, ldx, C, ldc, D, ldd):
        if M <= 0 or N <= 0:
            return
        ws = self._ws(200 << 20)
        self._chk(self.L.sqr_gemm_tn(M, N, K, alpha, X, ldx, C, ldc, 0.0, None, 0, D, ldd, ws.data_ptr(), ws.numel(),
                                     self._s()), "gemm_tn")

    def _gemm_nn(self, M, N, K, alpha, X, ldx, Y, ldy, beta, E, lde, D, ldd):
        if M <= 0 or N <= 0:
            return
        self._chk(self.L.sqr_gemm_nn(M, N, K, alpha, X, ldx, Y, ldy, beta, E, lde, D, ldd, self._s()), "gemm_nn")

    def tr_panel(self, S, lc, i0, m, k, w, bb, is_owner, Yg):
        """Owner: panel = work[i0:, sel] - Yg[i0:, :i0] Wg[:i0, sel] (randomized.py:304-306),
        then its Householder QR (:307) into the broadcast record."""
        self._select_panel_buffer(i0)
        mr = m - i0
        Y, taus, R11, st, rec, tail = self._panel_views(mr, bb)
        if is_owner:
            rec.zero_()
            LD = S.shape[1]
            base = S.data_ptr() + 8 * lc * LD
            if not hasattr(self, "Pn") or self.Pn.numel() < bb * mr:
                self.Pn = torch.empty(bb * m, dtype=torch.float64, device=self.dev)
            Pn = self.Pn[:bb * mr].view(bb, mr)
            if i0:
                self._gemm_nn(mr, w, i0, -1.0, Yg.data_ptr() + 8 * i0, m, base + 8 * m, LD, 1.0, base + 8 * i0, LD,
                              Pn.data_ptr(), mr)
            else:
                self._chk(self.L.sqr_copy_columns(base, LD, mr, None, Pn.data_ptr(), mr, None, w, self._s()), "panel")
            ws = self._ws(self.L.sqr_block_workspace(mr, 0, bb))
            self._chk(self.L.sqr_panel_factor(Pn.data_ptr(), mr, mr, w, Y.data_ptr(), mr, taus.data_ptr(), 1,
                                              st.data_ptr(), ws.data_ptr(), ws.numel(), self._s()), "panel")
            R11.copy_(Pn[:bb, :bb])
        return _Panel(0, Y, taus, None, R11, None, st)

    def tr_update(self, S, t0, i0, m, k, pan, bhat, Yg, lc):
        """Yg block, R11 into Rg (owner), then for this rank's trailing columns:
        G = Y2^T work - (Y2^T Y1) W1^T; Wg rows = T2^T G; R rows = work rows -
        Yg[i0:i0+bhat, :i0+bhat] Wg[:i0+bhat] (randomized.py:311-330)."""
        mr = m - i0
        LD = S.shape[1]
        Y = pan.Y                                   # (bb, mr): column c of Y2 is row c
        Yg[i0:i0 + bhat, i0:].copy_(Y[:bhat])
        if lc >= 0:                                 # Rg[i0:i0+bhat, panel] = triu(R11) on the owner
            R11 = torch.triu(pan.R11[:bhat, :bhat].T).T    # stored column-major: row index = column
            S[lc:lc + bhat, m + k + i0:m + k + i0 + bhat].copy_(R11)
        nloc = S.shape[0] - t0 if S.shape[0] > t0 else 0
        if nloc <= 0:
            return
        T2 = self.T.view(-1)[:bhat * bhat]
        wsb = self._ws(bhat * bhat * 8 + (200 << 20))
        self._chk(self.L.sqr_build_t(Y.data_ptr(), mr, mr, bhat, pan.taus.data_ptr(), T2.data_ptr(), bhat,
                                     wsb.data_ptr(), wsb.numel(), self._s()), "build_t")
        if not hasattr(self, "Gtr") or self.Gtr.numel() < bhat * (nloc + max(i0, 1)):
            self.Gtr = torch.empty(bhat * (S.shape[0] + k + 1), dtype=torch.float64, device=self.dev)
        G = self.Gtr[:bhat * nloc]
        C1 = self.Gtr[bhat * nloc:bhat * (nloc + max(i0, 1))]
        col = S.data_ptr() + 8 * t0 * LD
        self._gemm_tn(bhat, nloc, mr, 1.0, Y.data_ptr(), mr, col + 8 * i0, LD, G.data_ptr(), bhat)
        if i0:
            self._gemm_tn(bhat, i0, mr, 1.0, Y.data_ptr(), mr, Yg.data_ptr() + 8 * i0, m, C1.data_ptr(), bhat)
            self._gemm_nn(bhat, nloc, i0, -1.0, C1.data_ptr(), bhat, col + 8 * m, LD, 1.0, G.data_ptr(), bhat,
                          G.data_ptr(), bhat)
        self._gemm_tn(bhat, nloc, bhat, 1.0, T2.data_ptr(), bhat, G.data_ptr(), bhat, col + 8 * (m + i0), LD)
        self._gemm_nn(bhat, nloc, i0 + bhat, -1.0, Yg.data_ptr() + 8 * i0, m, col + 8 * m, LD, 1.0,
                      col + 8 * i0, LD, col + 8 * (m + k + i0), LD)

    # 6. sample update of my columns, written straight into the all-gather slab
    def sample_update_local(self, samp, A, s0, rel, i0, bb, pan, r_row0=None):
        """r_row0: storage row of the block's first R row (RQRCP: i0, in place;
        TRQRCP: the Rg rows of the stacked slab, m + k + i0)."""
        ell = samp.Bf.shape[1]
        nloc = len(rel)
        r_row0 = i0 if r_row0 is None else r_row0
        prepped = self.prep_done is not None
        if prepped:  # the overlapped prep wrote mbuf and may have set samp.st->stop
            self._cur().wait_event(self.prep_done)
            self.prep_done = None
        if nloc == 0:
            return self.slab[:0]
        ld = A.shape[1]
        if prepped and rel[-1] - rel[0] == nloc - 1 and s0 >= bb:
            # no gathers: the apply reads only S12 = Bf[:, b:] and R12 = R[:, b:]
            # (M = S11 R11^-1 came from the prep), so both are passed in place,
            # based b columns before my first trailing column (contiguous: a
            # world of one, or the last rank's tail)
            Sb = samp.Bf.data_ptr() + 8 * (int(rel[0]) - bb) * ell
            Rb = A.data_ptr() + 8 * ((s0 - bb) * ld + r_row0)
            # a world of one (NCCL path): straight into the replicated sample
            out = self.Bglob[i0 + bb:i0 + bb + nloc] if (self.symm is None and self._P == 1) else self.slab[:nloc]
            self._chk(self.L.sqr_sample_update_apply(Sb, ell, ell, Rb, ld, nloc, bb, out.data_ptr(), ell,
                                                     samp.st.data_ptr(), self.mbuf.data_ptr(), self._s()),
                      "sample_update")
            return out
        # Bf_loc = [S11 | Bf[:, rel]] and R_loc = [R11 | R12 of my columns]
        Bfl = self.Bfl[:bb + nloc]
        Bfl[:bb].copy_(samp.Bf[:bb])
        rel_d = self._idx(rel)
        self._chk(self.L.sqr_copy_columns(samp.Bf.data_ptr(), ell, ell, rel_d.data_ptr(),
                                          Bfl.data_ptr() + 8 * bb * ell, ell, None, nloc, self._s()), "gather S")
        Rl = self.Rl.view(-1)[:(bb + nloc) * bb].view(bb + nloc, bb)
        Rl[:bb].copy_(pan.R11)
        self._chk(self.L.sqr_copy_columns(A.data_ptr() + 8 * (s0 * ld + r_row0), ld, bb, None,
                                          Rl.data_ptr() + 8 * bb * bb, bb, None, nloc, self._s()), "gather R12")
        if prepped:  # M from the overlapped prep
            self._chk(self.L.sqr_sample_update_apply(Bfl.data_ptr(), ell, ell, Rl.data_ptr(), bb, nloc, bb,
                                                     self.slab.data_ptr(), ell, samp.st.data_ptr(),
                                                     self.mbuf.data_ptr(), self._s()), "sample_update")
        else:
            self._chk(self.L.sqr_sample_update_b(Bfl.data_ptr(), ell, ell, Rl.data_ptr(), bb, nloc, bb,
                                                 self.slab.data_ptr(), ell, samp.st.data_ptr(), self.mbuf.data_ptr(),
                                                 self._s()), "sample_update")
        return self.slab[:nloc]


# ----------------------------------------------------------------- bench
def local_giid(m: int, n: int, b: int, seed: int, lay: BlockCyclic, r: int, device, rows: int = 0) -> torch.Tensor:
    """This rank's columns of giid(m, n, seed) (column-major stream, rng.py:65-70)
    as (ncols, max(rows, m)) storage; rows beyond m are zero."""
    from . import _lib
    L = _lib.lib()
    nl = lay.n_local(r)
    ld = max(rows, m)
    A = torch.zeros((max(nl, 1), ld), dtype=torch.float64, device=device)
    j = 0
    for c in lay.blocks_of(r):
        w = min(b, n - c * b)
        L.sqr_gaussian(A.data_ptr() + 8 * j * ld, ld, m, w, seed, c * b * m, 0,
                       torch.cuda.current_stream(device).cuda_stream)
        j += w
    return A


class _OpsTimer:
    """SQR_DIST_TRACE=1: wraps every ops call with a device synchronisation and
    accumulates wall time per method (diagnostics only; perturbs timing)."""

    def __init__(self, ops, dev):
        import time
        self._ops, self._dev, self._t, self._time = ops, dev, {}, time

    def __getattr__(self, name):
        f = getattr(self._ops, name)
        if not callable(f):
            return f

        def wrapped(*a, **k):
            torch.cuda.synchronize(self._dev)
            t0 = self._time.perf_counter()
            out = f(*a, **k)
            torch.cuda.synchronize(self._dev)
            self._t[name] = self._t.get(name, 0.0) + self._time.perf_counter() - t0
            return out
        return wrapped

    def report(self):
        return {k: round(v * 1e3, 1) for k, v in sorted(self._t.items(), key=lambda kv: -kv[1])}


def bench_main(args, bench):
    """bench.py --gpus N under torchrun: strong scaling of C5 (n = 32768).

    ``bench`` is the bench.py module (metric, peak, config and clock helpers).
    Per rank: device time of the K timed steps with CUDA events between two
    barriers, max over ranks; e2e = the same call with this rank's columns
    uploaded from pinned host memory and its factored columns read back."""
    import json
    import os
    import time

    if "RANK" not in os.environ:  # --force-distributed without torchrun: a world of one
        os.environ.update({"RANK": "0", "LOCAL_RANK": "0", "WORLD_SIZE": "1", "MASTER_ADDR": "127.0.0.1",
                           "MASTER_PORT": os.environ.get("MASTER_PORT", "29531")})
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = SymmComm(None, dev) if getattr(args, "collectives", "nccl") == "symm" else TorchComm()
    from . import _lib
    L = _lib.lib()
    m = n = args.n
    b, p = args.b, args.p
    lay = BlockCyclic(n, b, comm.size)
    A0 = local_giid(m, n, b, 5, lay, comm.rank, dev, rows=m + 2 * b)  # + W rows (paired sweep)
    ops = GpuOps(dev, comm)
    tracer = None
    if os.environ.get("SQR_DIST_TRACE"):
        tracer = _OpsTimer(ops, dev)
        ops = tracer
    torch.cuda.synchronize()

    def step(A_src):
        A = A_src.clone()
        return rqrcp_block_cyclic(A, m, n, n, b, p, 0, comm, ops), A

    for _ in range(args.warmup):
        step(A0)
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = L.sqr_launch_count()
    L.sqr_profile_enable(20000 * max(1, args.steps))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            res, _ = step(A0)
        e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    launches = L.sqr_launch_count() - launches0
    prof = _lib.profile_collect()
    L.sqr_profile_enable(0)
    ms = comm.max(e0.elapsed_time(e1) / args.steps)
    gflop = bench.lapack_gflop(m, n)
    value = gflop / (ms / 1e3)
    # roofline of this rank's dominant GEMM class: its local share of the flops
    fl = bench.rqrcp_flops_by_kernel(m, n, n, b, p)
    dom = max(("gemm_tn", "gemm_nn"), key=lambda t: prof[t][0])
    share = lay.n_local(comm.rank) / n
    dom_ms = prof[dom][0] / args.steps
    ach_tf = fl[dom] * share / (dom_ms / 1e3) / 1e12 if dom_ms > 0 else None
    # e2e: pinned host columns in, factored columns out
    e2e = None
    if args.e2e_steps > 0:
        A_host = torch.empty_like(A0, device="cpu").pin_memory()
        A_host.copy_(A0)
        out_host = torch.empty_like(A_host).pin_memory()
        torch.cuda.synchronize()
        dist.barrier()
        ts = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            Ad = A_host.to(dev, non_blocking=True)
            r2, A_fact = step(Ad)
            out_host.copy_(A_fact, non_blocking=True)
            torch.cuda.synchronize()
            ts.append(comm.max(time.perf_counter() - t0))
        t_e2e = float(np.median(ts))
        e2e = {"value": gflop / t_e2e, "unit": "GFLOP/s", "h2d_bytes_per_step": int(A_host.numel() * 8),
               "d2h_bytes_per_step": int(out_host.numel() * 8), "ms_per_step": t_e2e * 1e3,
               "steps": args.e2e_steps, "api": "distributed.rqrcp_block_cyclic on this rank's pinned columns",
               "per_rank_bytes": True}
    clocks = clk.summary()
    if rank == 0:
        line = {"metric": bench.METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": comm.size,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(bench.base_config(args, f"column block-cyclic x{comm.size} "
                                                       f"({'symmetric-memory puts' if getattr(comm, 'symm', False) else 'NCCL'})"),
                               achieved_rank=res.achieved, l2="inputs larger than L2; no flush needed"),
                "roofline": {"bound": "tensor", "kernel": dom, "achieved": ach_tf, "peak": bench.PEAK_FP64_TFLOPS,
                             "unit": "TFLOP/s", "frac": (ach_tf / bench.PEAK_FP64_TFLOPS) if ach_tf else None,
                             "traffic": None, "peak_source": bench.PEAK_SOURCE, "rank": 0},
                "cpu_baseline": None, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks,
                "phases": {t: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
                           for t, v in prof.items() if v[1]}}
        if tracer is not None:
            line["host_trace_ms"] = tracer.report()
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


# ------------------------------------------------------------ public API
# The reference's call signatures (randomized.py:227, 250, 353) for a job of
# one process per GPU: every rank calls with the SAME full A (host array or
# tensor) and gets the same drop-in result object, assembled on every rank.
# Each rank uploads only its own block-cyclic columns.
_COMMS: dict = {}


def _comm(group, collectives="nccl", dev=None):
    """collectives="nccl": host-launched NCCL broadcast / all-gather;
    "symm": device-initiated puts into symmetric memory (SymmComm, csrc/peer.cu).
    A SymmComm (and its symmetric region) is kept per (group, device)."""
    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("distributed.rqrcp/trqrcp/tuxv need an initialised torch.distributed process group "
                           "(one process per GPU, backend 'nccl')")
    if collectives == "nccl":
        return TorchComm(group)
    if collectives != "symm":
        raise ValueError("collectives must be 'nccl' or 'symm'")
    key = (id(group), str(dev))
    if key not in _COMMS:
        _COMMS[key] = SymmComm(group, dev)
    return _COMMS[key]


def _local_slab(A, cols: np.ndarray, m: int, rows: int, dev) -> torch.Tensor:
    """This rank's columns of the caller's full m x n A as (ncols, rows) device
    storage (rows >= m; the extra rows are zero), plus the input contract of
    validation.check_matrix on them (validation.py:21-38)."""
    from . import _lib
    nl = int(cols.size)
    S = torch.zeros((max(nl, 1), rows), dtype=torch.float64, device=dev)
    if nl:
        if isinstance(A, torch.Tensor):
            src = A.detach().to(device=dev, dtype=torch.float64)
            S[:nl, :m] = src[:, torch.as_tensor(cols, device=dev)].T
        else:
            host = np.asarray(A, dtype=np.float64)[:, cols]
            S[:nl, :m].copy_(torch.from_numpy(np.ascontiguousarray(host.T)))
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    if nl and m:
        _lib.check(_lib.lib().sqr_copy_check(S.data_ptr(), rows, m, nl, None, 0, cnt.data_ptr(),
                                             torch.cuda.current_stream(dev).cuda_stream), "sqr_copy_check")
    return S, cnt


def _shape_of(A):
    if isinstance(A, torch.Tensor):
        if A.dim() != 2:
            raise ValueError(f"A must be 2-dimensional, got ndim={A.dim()}")
        return tuple(int(x) for x in A.shape)
    arr = np.asarray(A)
    if arr.ndim != 2:
        raise ValueError(f"A must be 2-dimensional, got ndim={arr.ndim}")
    return arr.shape


def _omega_arg(omega, ell, m, seed):
    """None / "device": drawn on the device by every rank (same stream, same
    bits); "host": the reference's NumPy recipe; else an explicit l x m array."""
    if omega is None or (isinstance(omega, str) and omega == "device"):
        return None
    if isinstance(omega, str):
        if omega != "host":
            raise ValueError("omega must be 'device', 'host' or an l x m array")
        from .rng import host_omega
        return host_omega(ell, m, seed)
    om = omega.detach().cpu().numpy() if isinstance(omega, torch.Tensor) else np.asarray(omega, dtype=np.float64)
    if om.shape != (ell, m):
        raise ValueError(f"omega must have shape ({ell}, {m}), got {om.shape}")
    return om


def _gather_columns(S: torch.Tensor, lay: BlockCyclic, comm, rows: int, dev):
    """All ranks' slabs into one (rows x n) column-major matrix in global column order."""
    from . import _lib
    from ._dev import ColMajor
    nmax = lay.n_local_max()
    mine = torch.zeros((max(nmax, 1), rows), dtype=torch.float64, device=dev)
    nl = lay.n_local(comm.rank)
    if nl:
        mine[:nl] = S[:nl, :rows]
    parts = comm.all_gather(mine)
    W = ColMajor.empty(rows, lay.n, dev, ld=rows)
    s = torch.cuda.current_stream(dev).cuda_stream
    for q, part in enumerate(parts):
        g = lay.global_of_local(q)
        if g.size:
            gi = torch.tensor(g, device=dev)
            _lib.check(_lib.lib().sqr_copy_columns(part.data_ptr(), rows, rows, None, W.ptr, rows, gi.data_ptr(),
                                                   int(g.size), s), "gather columns")
    return W


def _prologue(A, k, b, p, comm, dev):
    from . import factor as F
    m, n = _shape_of(A)
    F._check_block_args(m, n, k, b, p)
    return m, n


def _check_finite_all(cnt, comm):
    if comm.max(float(cnt.item())) > 0:
        raise ValueError("A contains non-finite entries")


def rqrcp(A, k: int, b: int = 32, p: int = 8, seed: int = 0, omega=None, group=None, device=None,
          collectives: str = "nccl"):
    """Multi-GPU drop-in of randomized.rqrcp (randomized.py:227-229): column
    block-cyclic over the process group, NCCL.  Returns the reference's
    PivotedFactorization (R, perm, blocks, achieved_rank, counters) on every
    rank."""
    from . import factor as F
    from ._dev import require_cuda
    dev = require_cuda(device)
    comm = _comm(group, collectives, dev)
    m, n = _prologue(A, k, b, p, comm, dev)
    ell = b + p
    if k == 0 or ell >= m:   # empty / the deterministic l >= m fallback (randomized.py:172-174): replicated
        return F.rqrcp(A, k, b=b, p=p, seed=seed, omega=omega)
    lay = BlockCyclic(n, b, comm.size)
    # rows [m, m + 2b): W_P | W_J of the paired second sweep (they move with the columns)
    S, bad = _local_slab(A, lay.global_of_local(comm.rank), m, m + 2 * b, dev)
    _check_finite_all(bad, comm)
    res = rqrcp_block_cyclic(S, m, n, k, b, p, seed, comm, GpuOps(dev, comm), omega=_omega_arg(omega, ell, m, seed))
    W = _gather_columns(S, lay, comm, m, dev)
    ach = res.achieved
    pf = F.PivotedFactorization(m, n, None, None, None, ach, res.counters)
    pf._Rd_fn = lambda: F._upper_rows(W, ach)
    pf._permd = torch.as_tensor(res.perm, device=dev)
    taus = torch.as_tensor(np.asarray(res.taus, dtype=np.float64), device=dev)
    widths = [(J * b, min(b, ach - J * b)) for J in range(res.nblocks)]
    pf._blocks_fn = lambda: F._packed_blocks(W, taus, None, b, widths, m)
    pf._work = W
    return pf


def _trqrcp_dist(A, k, b, p, seed, allow_large_k, omega, group, device, collectives="nccl"):
    from . import factor as F
    from ._dev import ColMajor, require_cuda
    dev = require_cuda(device)
    comm = _comm(group, collectives, dev)
    m, n = _prologue(A, k, b, p, comm, dev)
    if not allow_large_k and k > min(m, n) // 2:
        raise ValueError("trqrcp targets k <= min(m, n)/2; pass allow_large_k=True to override")
    ell = b + p
    if k == 0 or ell >= m:
        return None, None, None, dev, comm, m, n
    lay = BlockCyclic(n, b, comm.size)
    rows = m + 2 * k
    S, bad = _local_slab(A, lay.global_of_local(comm.rank), m, rows, dev)
    _check_finite_all(bad, comm)
    res = trqrcp_block_cyclic(S, m, n, k, b, p, seed, comm, GpuOps(dev, comm), omega=_omega_arg(omega, ell, m, seed))
    SW = _gather_columns(S, lay, comm, rows, dev)
    ach = res.achieved
    tf = F.TruncatedFactorization(m, n, None, None, None, ach, res.counters)
    Rv = ColMajor(SW.t[:, m + k:], k, n, SW.ld)
    tf._Rd = F._upper_rows(Rv, ach)
    wt = torch.empty((ach, n), dtype=torch.float64, device=dev)
    if ach:
        from . import _lib
        _lib.check(_lib.lib().sqr_transpose(SW.ptr + 8 * m, SW.ld, ach, n, wt.data_ptr(), n, 0,
                                            torch.cuda.current_stream(dev).cuda_stream), "sqr_transpose")
    tf._w_td = wt
    tf._permd = torch.as_tensor(res.perm, device=dev)
    taus = torch.as_tensor(np.asarray(res.taus, dtype=np.float64), device=dev)
    widths = [(J * b, min(b, ach - J * b)) for J in range(res.nblocks)]
    Yg = ColMajor(res.Yg, m, k, m)
    tf._blocks_fn = lambda: F._packed_blocks(Yg, taus, None, b, widths, m)
    return tf, S, lay, dev, comm, m, n


def trqrcp(A, k: int, b: int = 32, p: int = 8, seed: int = 0, allow_large_k: bool = False, omega=None,
           group=None, device=None, collectives: str = "nccl"):
    """Multi-GPU drop-in of randomized.trqrcp (randomized.py:250-341); the
    TruncatedFactorization (R, w_t, perm, blocks, counters) on every rank."""
    from . import factor as F
    tf, *_ = _trqrcp_dist(A, k, b, p, seed, allow_large_k, omega, group, device, collectives)
    if tf is None:
        return F.trqrcp(A, k, b=b, p=p, seed=seed, allow_large_k=allow_large_k, omega=omega)
    return tf


def tuxv(A, k: int, j_max: int = 1, b: int = 32, p: int = 8, seed: int = 0, refine_sigma: bool = False,
         allow_large_k: bool = False, omega=None, group=None, device=None, collectives: str = "nccl"):
    """Multi-GPU drop-in of randomized.tuxv (randomized.py:353-406): the
    distributed TRQRCP, then the QLP flip-flop with A's products formed from
    the local slabs -- A V_k as a sum of per-rank partials (all-reduce of the
    m x k partial Z), (U^T A)^T as disjoint row blocks
    (all-reduce of an n x k matrix that each rank fills only at its columns)."""
    from . import factor as F
    from . import _lib
    from ._dev import ColMajor
    if j_max < 1:
        raise ValueError("j_max must be >= 1")
    tf, S, lay, dev, comm, m, n = _trqrcp_dist(A, k, b, p, seed, allow_large_k, omega, group, device, collectives)
    if tf is None:
        return F.tuxv(A, k, j_max=j_max, b=b, p=p, seed=seed, refine_sigma=refine_sigma,
                      allow_large_k=allow_large_k, omega=omega)
    L = _lib.lib()
    rows = S.shape[1]
    nl = lay.n_local(comm.rank)
    Wloc = ColMajor(S, m, nl, rows)                            # this rank's columns of A P (work rows)
    orig = torch.as_tensor(tf.perm[lay.global_of_local(comm.rank)], device=dev)   # their original columns

    def s():
        return torch.cuda.current_stream(dev).cuda_stream

    def a_times(Vk):
        Vl = ColMajor.empty(max(nl, 1), Vk.n, dev)
        if nl:
            _lib.check(L.sqr_gather_rows(Vk.ptr, Vk.ld, nl, Vk.n, orig.data_ptr(), Vl.ptr, Vl.ld, s()), "gather")
            Vl.m = nl
            Z = F.gemm_nn(Wloc, Vl)
        else:
            Z = ColMajor.empty(m, Vk.n, dev, zero=True)
        dist.all_reduce(Z.t, group=comm.group)
        return Z

    def at_times(Uk):
        Z = ColMajor.empty(n, Uk.n, dev, zero=True)
        if nl:
            Zt = F._transpose(F.gemm_tn(Uk, Wloc))            # nl x kh
            _lib.check(L.sqr_scatter_rows(Zt.ptr, Zt.ld, nl, Uk.n, orig.data_ptr(), Z.ptr, Z.ld, s()), "scatter")
        dist.all_reduce(Z.t, group=comm.group)
        return Z

    return F._qlp(tf, m, n, b, j_max, refine_sigma, a_times, at_times, dev)

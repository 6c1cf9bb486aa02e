"""Multi-process (gloo, CPU) test of the column block-cyclic RQRCP
orchestration (paper_2008_04447_b200/distributed.py): world sizes 2 and 3
must reproduce the single-process oracle (identical permutation, counters,
achieved rank; R to 1e-10)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import gauss


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _matrix(m, n, rr):
    A = gauss(m, n, 17)
    if rr > 0:  # rank-deficient: the sample floor stops the loop behind a pending block
        A = np.asfortranarray(gauss(m, rr, 18) @ gauss(rr, n, 19))
    elif rr < 0:  # -rr independent columns then exact zeros: a short panel (bhat < b) settles lazily
        A = np.zeros((m, n), order="F")
        A[:, :-rr] = gauss(m, -rr, 18)
    return A


def _worker(rank, world, port, m, n, k, b, p, seed, q, rr=0, algo="rqrcp"):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_numpy_ops import NumpyOps
        from paper_2008_04447_b200.distributed import (BlockCyclic, TorchComm, rqrcp_block_cyclic,
                                                       trqrcp_block_cyclic)
        A = _matrix(m, n, rr)
        lay = BlockCyclic(n, b, world)
        g = lay.global_of_local(rank)
        if algo == "trqrcp":   # stacked [work; Wg; Rg] columns
            A_loc = torch.zeros((g.size, m + 2 * k), dtype=torch.float64)
            A_loc[:, :m] = torch.from_numpy(np.ascontiguousarray(A[:, g].T))
            res = trqrcp_block_cyclic(A_loc, m, n, k, b, p, seed, TorchComm(), NumpyOps())
            m = m + 2 * k      # gather the whole stacked slab below
        elif algo == "rqrcp_paired":   # storage rows [m, m + 2b): the paired second sweep's W_P | W_J
            A_loc = torch.zeros((g.size, m + 2 * b), dtype=torch.float64)
            A_loc[:, :m] = torch.from_numpy(np.ascontiguousarray(A[:, g].T))
            res = rqrcp_block_cyclic(A_loc, m, n, k, b, p, seed, TorchComm(), NumpyOps())
        else:
            A_loc = torch.from_numpy(np.ascontiguousarray(A[:, g].T))
            res = rqrcp_block_cyclic(A_loc, m, n, k, b, p, seed, TorchComm(), NumpyOps())
        parts = [torch.zeros((max(lay.n_local(r) for r in range(world)), m), dtype=torch.float64)
                 for _ in range(world)]
        mine = torch.zeros_like(parts[0])
        mine[:A_loc.shape[0]] = A_loc[:, :m]
        dist.all_gather(parts, mine)
        if rank == 0:
            W = np.zeros((m, n))
            for r in range(world):
                gr = lay.global_of_local(r)
                W[:, gr] = parts[r][:gr.size].numpy().T
            q.put((res.achieved, res.perm, W, [res.counters.trailing_passes, res.counters.blas3_volume],
                   res.reason))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,k,b,p,rr", [(2, 90, 70, 70, 8, 4, 0), (3, 120, 100, 60, 16, 8, 0),
                                                (2, 64, 80, 64, 8, 8, 0), (2, 90, 70, 70, 8, 4, 29),
                                                (3, 100, 90, 90, 16, 4, 37), (2, 90, 70, 70, 8, 4, -29),
                                                (4, 130, 150, 120, 8, 8, 0), (8, 140, 200, 136, 8, 4, 0)])
def test_block_cyclic_matches_oracle(world, m, n, k, b, p, rr):
    _check_block_cyclic(world, m, n, k, b, p, rr, "rqrcp")


@pytest.mark.parametrize("world,m,n,k,b,p,rr", [(2, 90, 70, 70, 8, 4, 0), (3, 120, 100, 60, 16, 8, 0),
                                                (2, 90, 70, 70, 8, 4, 29), (3, 100, 90, 90, 16, 4, 37),
                                                (2, 90, 70, 70, 8, 4, -29), (4, 130, 150, 120, 8, 8, 0),
                                                (8, 140, 200, 136, 8, 4, 0), (2, 64, 80, 40, 8, 8, 0)])
def test_block_cyclic_paired_matches_oracle(world, m, n, k, b, p, rr):
    """The paired second sweep (distributed.rqrcp_block_cyclic with W rows in
    the storage): identical permutation / counters and R to 1e-10, including
    rank-deficient (short / zero panel, sample floor) exits with a deferred
    block pending."""
    _check_block_cyclic(world, m, n, k, b, p, rr, "rqrcp_paired")


def _check_block_cyclic(world, m, n, k, b, p, rr, algo):
    from oracle import port as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, b, p, 5, q, rr, algo)) for r in range(world)]
    for pr in procs:
        pr.start()
    achieved, perm, W, cnt, reason = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    A = _matrix(m, n, rr)
    ref = O.rqrcp(A, k, b=b, p=p, seed=5)
    R = np.triu(W[:achieved, :])
    dr = np.abs(np.diag(ref.R[:ref.achieved_rank, :ref.achieved_rank]))
    floor = 1e-10 * dr[0] if dr.size else 0.0
    sig = int(np.count_nonzero(dr > floor))
    if algo == "rqrcp_paired" and sig < ref.achieved_rank:
        # pivots among columns already at the noise floor are rounding-level
        # near-ties (the merged sweep rounds differently from the reference's
        # per-block update): everything above the noise floor must agree
        d = np.abs(np.diag(R[:achieved, :achieved]))
        assert np.all(d[sig:] <= floor)
        assert np.array_equal(perm[:sig], ref.perm[:sig])
        assert np.all(np.abs(d[:sig] - dr[:sig]) <= 1e-10 * dr[:sig])
        return
    assert achieved == ref.achieved_rank
    assert np.array_equal(perm, ref.perm)
    assert cnt == [ref.counters.trailing_passes, ref.counters.blas3_volume]
    assert np.abs(R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()


def test_layout_roundtrip():
    from paper_2008_04447_b200.distributed import BlockCyclic
    for n, b, P in [(100, 8, 3), (128, 128, 4), (7, 2, 5)]:
        lay = BlockCyclic(n, b, P)
        seen = np.concatenate([lay.global_of_local(r) for r in range(P)])
        assert np.array_equal(np.sort(seen), np.arange(n))
        for r in range(P):
            g = lay.global_of_local(r)
            assert np.all(lay.owner(g) == r)
            assert np.array_equal(lay.local_index(g), np.arange(g.size))
        assert sum(lay.n_local(r) for r in range(P)) == n


def test_move_plan_is_a_simultaneous_permutation():
    """distributed.move_plan (used by both backends) applied rank by rank equals
    the single-process column permutation, for random move sets."""
    from paper_2008_04447_b200.distributed import BlockCyclic, move_plan
    rng = np.random.default_rng(3)
    for n, b, P in [(64, 8, 3), (100, 16, 4), (40, 4, 2)]:
        lay = BlockCyclic(n, b, P)
        for _ in range(20):
            i0 = int(rng.integers(0, n - b))
            k = int(rng.integers(1, b + 1))
            # a block-style permutation: positions i0..i0+k receive k distinct sources
            src = rng.choice(np.arange(i0, n), size=k, replace=False)
            perm = np.arange(n)
            for j, s in enumerate(src):
                perm[[i0 + j, s]] = perm[[s, i0 + j]]
            changed = np.nonzero(perm != np.arange(n))[0]
            pd, ps = changed, perm[changed]
            cols = np.arange(n, dtype=np.float64) * 10.0
            want = cols[perm]
            local = [cols[lay.global_of_local(r)].copy() for r in range(P)]
            plans = [move_plan(ps, pd, lay, r) for r in range(P)]
            packed = [local[r][p.pack].copy() for r, p in enumerate(plans)]
            new = [x.copy() for x in local]
            for r, p in enumerate(plans):
                new[r][p.local_dst] = packed[r][p.local_rows]
                for q, dst in p.recv.items():
                    new[r][dst] = packed[q][plans[q].send[r]]
            got = np.empty(n)
            for r in range(P):
                got[lay.global_of_local(r)] = new[r]
            assert np.array_equal(got, want)


@pytest.mark.parametrize("world,m,n,k,b,p,rr", [(2, 90, 70, 30, 8, 4, 0), (3, 150, 120, 48, 16, 8, 0),
                                                (4, 130, 150, 40, 8, 8, 0), (8, 120, 200, 64, 8, 4, 0),
                                                (2, 90, 70, 35, 8, 4, 29), (3, 100, 90, 45, 8, 4, -21)])
def test_trqrcp_block_cyclic_matches_oracle(world, m, n, k, b, p, rr):
    """Distributed TRQRCP (distributed.trqrcp_block_cyclic): identical
    permutation / counters, and R and W^T rows to 1e-10 of the single-process
    oracle (randomized.py:250-341), including exits behind a short panel."""
    from oracle import port as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, b, p, 5, q, rr, "trqrcp"))
             for r in range(world)]
    for pr in procs:
        pr.start()
    achieved, perm, S, cnt, reason = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    A = _matrix(m, n, rr)
    ref = O.trqrcp(A, k, b=b, p=p, seed=5, allow_large_k=True)
    assert achieved == ref.achieved_rank
    assert np.array_equal(perm, ref.perm)
    assert cnt == [ref.counters.trailing_passes, ref.counters.blas3_volume]
    Wt = S[m:m + achieved, :]
    R = np.triu(S[m + k:m + k + achieved, :])
    assert np.abs(R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()
    assert np.abs(Wt - ref.w_t).max() <= 1e-10 * max(np.abs(ref.w_t).max(), 1e-300)
    # the stacked work rows are only permuted, never updated (randomized.py:278)
    assert np.array_equal(S[:m, :], A[:, perm])

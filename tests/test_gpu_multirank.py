"""The multi-GPU path with REAL peers (NCCL point-to-point column moves,
owner-only panels, the symmetric-memory puts): world size 2..4 on as many
GPUs as the box has, one process per GPU, against the single-process oracle.
Skipped on a one-GPU box (this pool's gpurun gives one GPU; the orchestration
logic with peers is covered on CPU by tests/test_distributed_gloo.py)."""
import os
import socket

import numpy as np
import pytest

from conftest import gauss

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, collectives):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        import paper_2008_04447_b200.distributed as D
        out = {}
        A = gauss(900, 700, 11)
        pf = D.rqrcp(A, 700, b=32, p=8, seed=0, omega="host", collectives=collectives)
        out["rqrcp"] = (pf.perm, pf.R, pf.achieved_rank)
        L = np.asfortranarray(gauss(600, 61, 12) @ gauss(61, 500, 13))      # rank exhaustion mid-block
        pl = D.rqrcp(L, 500, b=16, p=8, seed=1, omega="host", collectives=collectives)
        out["lowrank"] = (pl.perm, pl.R, pl.achieved_rank)
        tf = D.trqrcp(A, 96, b=32, p=8, seed=2, omega="host", collectives=collectives)
        out["trqrcp"] = (tf.perm, tf.w_t, tf.achieved_rank)
        x = D.tuxv(A, 20, b=8, p=8, seed=3, omega="host", collectives=collectives)
        out["tuxv"] = (x.reconstruct(), x.achieved_rank)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("collectives", ["nccl", "symm"])
def test_multi_gpu_matches_oracle(collectives):
    from oracle import port as O
    world = min(4, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, collectives)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = gauss(900, 700, 11)
    ref = O.rqrcp(A, 700, b=32, p=8, seed=0)
    perm, R, ach = out["rqrcp"]
    assert ach == ref.achieved_rank and np.array_equal(perm, ref.perm)
    assert np.abs(R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()
    L = np.asfortranarray(gauss(600, 61, 12) @ gauss(61, 500, 13))
    refl = O.rqrcp(L, 500, b=16, p=8, seed=1)
    perm, R, ach = out["lowrank"]
    assert ach == refl.achieved_rank
    assert np.array_equal(perm[:ach], refl.perm[:ach])
    tref = O.trqrcp(A, 96, b=32, p=8, seed=2)
    perm, wt, ach = out["trqrcp"]
    assert np.array_equal(perm, tref.perm)
    assert np.abs(wt - tref.w_t).max() <= 1e-10 * np.abs(tref.w_t).max()
    xref = O.tuxv(A, 20, b=8, p=8, seed=3)
    rec, ach = out["tuxv"]
    assert np.abs(rec - xref.reconstruct()).max() <= 1e-9 * np.abs(A).max()

"""GpuOps + NCCL backend of the block-cyclic driver on one B200 (world size 1:
every step of the multi-GPU path except the peer traffic, which the gloo test
covers).  Must match the single-GPU driver and the oracle."""
import socket

import numpy as np
import pytest

from conftest import gauss
from oracle import port as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_2008_04447_b200 as G  # noqa: E402
from paper_2008_04447_b200.distributed import GpuOps, TorchComm, rqrcp_block_cyclic  # noqa: E402


@pytest.fixture(scope="module")
def nccl1():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=dev)
    yield dev
    dist.destroy_process_group()


def _slab(A, m, rows, dev):
    """(ncols, rows) storage, rows [m, rows) zero: rows >= m + 2b turn on the
    paired second sweep (W_P | W_J rows)."""
    S = torch.zeros((A.shape[1], rows), dtype=torch.float64)
    S[:, :m] = torch.from_numpy(np.ascontiguousarray(A.T))
    return S.to(dev)


@pytest.mark.parametrize("plan", [False, True])
@pytest.mark.parametrize("paired", [False, True])
@pytest.mark.parametrize("m,n,k,b,p", [(600, 500, 500, 32, 8), (2000, 700, 300, 64, 8), (300, 257, 257, 16, 4)])
def test_block_cyclic_gpu_world1(nccl1, m, n, k, b, p, paired, plan):
    """plan=False: a world of one applies the sample QRCP's device move list
    directly; plan=True forces the P2P path (move plan, pack, exchange, unpack)."""
    dev = nccl1
    A = gauss(m, n, 3)
    om = O.gauss_matrix(b + p, m, 11)
    A_loc = _slab(A, m, m + 2 * b if paired else m, dev)
    ops = GpuOps(dev)
    ops.plan_moves = plan
    res = rqrcp_block_cyclic(A_loc, m, n, k, b, p, 11, TorchComm(), ops, omega=om)
    ref = O.rqrcp(A, k, b=b, p=p, seed=11)
    assert res.achieved == ref.achieved_rank
    assert np.array_equal(res.perm, ref.perm)
    W = A_loc[:, :m].cpu().numpy().T
    R = np.triu(W[:res.achieved, :])
    assert np.abs(R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()
    assert [res.counters.trailing_passes, res.counters.blas3_volume] == \
        [ref.counters.trailing_passes, ref.counters.blas3_volume]
    single = G.rqrcp(A, k, b=b, p=p, seed=11, omega=om)
    assert np.array_equal(single.perm, res.perm)


@pytest.mark.parametrize("paired", [False, True])
@pytest.mark.parametrize("kind", ["short_panel", "lowrank"])
def test_block_cyclic_gpu_lazy_exits(nccl1, kind, paired):
    """Early exits settled lazily (the panel tail read with the next block's
    sample record): a short panel and a sample-floor stop behind a pending block."""
    dev = nccl1
    m, n, b, p = 300, 200, 16, 8
    if kind == "short_panel":
        A = np.zeros((m, n), order="F")
        A[:, :53] = gauss(m, 53, 4)          # 3 full blocks + a 5-wide one
    else:
        A = np.asfortranarray(gauss(m, 61, 5) @ gauss(61, n, 6))
    om = O.gauss_matrix(b + p, m, 13)
    A_loc = _slab(A, m, m + 2 * b if paired else m, dev)
    res = rqrcp_block_cyclic(A_loc, m, n, n, b, p, 13, TorchComm(), GpuOps(dev), omega=om)
    ref = O.rqrcp(A, n, b=b, p=p, seed=13)
    assert res.achieved == ref.achieved_rank
    assert [res.counters.trailing_passes, res.counters.blas3_volume] == \
        [ref.counters.trailing_passes, ref.counters.blas3_volume]
    W = A_loc[:, :m].cpu().numpy().T
    R = np.triu(W[:res.achieved, :])
    d = np.nonzero(res.perm != ref.perm)[0]
    if d.size:  # documented near-tie: pivots among columns already at the noise floor
        j, dr = int(d[0]), np.abs(ref.r_diag)
        assert j >= res.achieved or dr[j] <= 1e-10 * dr[0]
        assert np.abs(np.abs(np.diag(R))[:j] - dr[:j]).max() <= 1e-10 * dr[0]
        return
    assert np.abs(R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()


@pytest.mark.parametrize("m,n,k,b,p", [(600, 500, 120, 32, 8), (1500, 900, 200, 64, 8), (300, 257, 90, 16, 4)])
def test_trqrcp_block_cyclic_gpu_world1(nccl1, m, n, k, b, p):
    """trqrcp_block_cyclic on GpuOps + NCCL (stacked [work; Wg; Rg] slab)."""
    from paper_2008_04447_b200.distributed import trqrcp_block_cyclic
    dev = nccl1
    A = gauss(m, n, 8)
    om = O.gauss_matrix(b + p, m, 11)
    S = torch.zeros((n, m + 2 * k), dtype=torch.float64, device=dev)
    S[:, :m] = torch.from_numpy(np.ascontiguousarray(A.T)).to(dev)
    res = trqrcp_block_cyclic(S, m, n, k, b, p, 11, TorchComm(), GpuOps(dev), omega=om)
    ref = O.trqrcp(A, k, b=b, p=p, seed=11, allow_large_k=True)
    assert res.achieved == ref.achieved_rank
    assert np.array_equal(res.perm, ref.perm)
    assert [res.counters.trailing_passes, res.counters.blas3_volume] == \
        [ref.counters.trailing_passes, ref.counters.blas3_volume]
    W = S.cpu().numpy().T
    R = np.triu(W[m + k:m + k + res.achieved])
    assert np.abs(R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()
    assert np.abs(W[m:m + res.achieved] - ref.w_t).max() <= 1e-10 * np.abs(ref.w_t).max()
    assert np.array_equal(W[:m], A[:, ref.perm])


def test_public_multi_gpu_api_world1(nccl1):
    """distributed.rqrcp / trqrcp / tuxv (the reference's signatures, one
    process per GPU) return the drop-in result objects: same pivots, R, w_t,
    blocks and counters as the oracle, methods (residual, Q columns) working."""
    import paper_2008_04447_b200.distributed as D
    A = gauss(700, 600, 21)
    pf = D.rqrcp(A, 600, b=32, p=8, seed=0, omega="host")
    ref = O.rqrcp(A, 600, b=32, p=8, seed=0)
    assert pf.achieved_rank == ref.achieved_rank and np.array_equal(pf.perm, ref.perm)
    assert np.abs(pf.R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()
    assert len(pf.blocks) == len(ref.blocks)
    assert [pf.counters.trailing_passes, pf.counters.blas3_volume] == \
        [ref.counters.trailing_passes, ref.counters.blas3_volume]
    assert pf.rel_residual(A) <= 1e-12
    Q = pf.q_columns()
    assert np.abs(Q.T @ Q - np.eye(Q.shape[1])).max() <= 1e-12
    tf = D.trqrcp(A, 96, b=32, p=8, seed=1, omega="host")
    tref = O.trqrcp(A, 96, b=32, p=8, seed=1)
    assert np.array_equal(tf.perm, tref.perm)
    assert np.abs(tf.R - tref.R).max() <= 1e-10 * np.abs(tref.R).max()
    assert np.abs(tf.w_t - tref.w_t).max() <= 1e-10 * np.abs(tref.w_t).max()
    assert abs(tf.rel_residual(A, 96) - tref.rel_residual(A, 96)) <= 1e-10 * tref.rel_residual(A, 96)
    for j_max in (1, 2):
        x = D.tuxv(A, 24, j_max=j_max, b=8, p=8, seed=2, omega="host")
        xref = O.tuxv(A, 24, j_max=j_max, b=8, p=8, seed=2)
        assert np.abs(x.reconstruct() - xref.reconstruct()).max() <= 1e-9 * np.abs(A).max()
        assert [x.counters.trailing_passes, x.counters.blas3_volume] == \
            [xref.counters.trailing_passes, xref.counters.blas3_volume]
    with pytest.raises(ValueError, match="non-finite"):
        B = A.copy()
        B[3, 4] = np.nan
        D.rqrcp(B, 10, b=8, p=4)


def test_peer_put_kernels_fake_peers():
    """csrc/peer.cu with P "peers" that are buffers of this one GPU (the same
    pointer arrays a symmetric-memory rendezvous provides): every peer copy
    receives the bytes / the scattered columns, every peer flag the epoch,
    the arrival counter returns to zero, and the wait passes once the flags
    carry the epoch."""
    from paper_2008_04447_b200 import _lib
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream().cuda_stream
    P, nbytes = 4, 1 << 20
    src = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=dev)
    dst = [torch.zeros(nbytes + 4096, dtype=torch.uint8, device=dev) for _ in range(P)]
    flags = [torch.zeros(8, dtype=torch.int64, device=dev) for _ in range(P)]
    dptr = torch.tensor([d.data_ptr() for d in dst], dtype=torch.int64, device=dev)
    fptr = torch.tensor([f.data_ptr() for f in flags], dtype=torch.int64, device=dev)
    ctr = torch.zeros(4, dtype=torch.int32, device=dev)
    for ep in (1, 2):
        _lib.check(L.sqr_peer_put(src.data_ptr(), nbytes, dptr.data_ptr(), 4096, P, fptr.data_ptr(), 3, ep,
                                  ctr.data_ptr(), s))
        _lib.check(L.sqr_peer_wait(flags[2].data_ptr() + 8 * 3, 1, ep, s))
        torch.cuda.synchronize()
        for q in range(P):
            assert torch.equal(dst[q][4096:], src) and int(flags[q][3]) == ep
        assert int(ctr[0]) == 0
    # put_columns: 3 local columns of a 40-row slab -> global positions 5, 1, 9 of every replica
    ell, n = 40, 12
    slab = torch.randn((3, ell), dtype=torch.float64, device=dev)
    didx = torch.tensor([5, 1, 9], dtype=torch.int64, device=dev)
    reps = [torch.zeros((n, ell), dtype=torch.float64, device=dev) for _ in range(P)]
    rptr = torch.tensor([r.data_ptr() for r in reps], dtype=torch.int64, device=dev)
    _lib.check(L.sqr_peer_put_columns(slab.data_ptr(), ell, ell, 3, didx.data_ptr(), rptr.data_ptr(), ell, P,
                                      fptr.data_ptr(), 5, 7, ctr.data_ptr(), s))
    _lib.check(L.sqr_peer_wait(flags[0].data_ptr(), 8, 0, s))
    torch.cuda.synchronize()
    for q in range(P):
        assert torch.equal(reps[q][[5, 1, 9]], slab) and int(reps[q].abs().sum(1).count_nonzero()) == 3
        assert int(flags[q][5]) == 7


@pytest.mark.parametrize("collectives", ["nccl", "symm"])
def test_public_api_symmetric_collectives_world1(nccl1, collectives):
    """The public multi-GPU entry points with the device-initiated collectives
    (SymmComm over torch symmetric memory) match the NCCL path bitwise."""
    import paper_2008_04447_b200.distributed as D
    A = gauss(500, 420, 31)
    pf = D.rqrcp(A, 420, b=32, p=8, seed=0, omega="host", collectives=collectives)
    ref = O.rqrcp(A, 420, b=32, p=8, seed=0)
    assert np.array_equal(pf.perm, ref.perm)
    assert np.abs(pf.R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()
    tf = D.trqrcp(A, 64, b=16, p=8, seed=1, omega="host", collectives=collectives)
    tref = O.trqrcp(A, 64, b=16, p=8, seed=1)
    assert np.array_equal(tf.perm, tref.perm)
    assert np.abs(tf.w_t - tref.w_t).max() <= 1e-10 * np.abs(tref.w_t).max()
    if collectives == "symm":
        nc = D.rqrcp(A, 420, b=32, p=8, seed=0, omega="host", collectives="nccl")
        assert np.array_equal(nc.perm, pf.perm) and np.array_equal(nc.R, pf.R)

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
from paper_2008_04447_b200.distributed import BlockCyclic, GpuOps, TorchComm, rqrcp_block_cyclic  # noqa: E402


@pytest.fixture(scope="module")
def nccl1():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=dev)
    yield dev
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n,k,b,p", [(600, 500, 500, 32, 8), (2000, 700, 300, 64, 8), (300, 257, 257, 16, 4)])
def test_block_cyclic_gpu_world1(nccl1, m, n, k, b, p):
    dev = nccl1
    A = gauss(m, n, 3)
    om = O.gauss_matrix(b + p, m, 11)
    lay = BlockCyclic(n, b, 1)
    A_loc = torch.from_numpy(np.ascontiguousarray(A.T)).to(dev)
    res = rqrcp_block_cyclic(A_loc, m, n, k, b, p, 11, TorchComm(), GpuOps(dev), omega=om)
    ref = O.rqrcp(A, k, b=b, p=p, seed=11)
    assert res.achieved == ref.achieved_rank
    assert np.array_equal(res.perm, ref.perm)
    W = A_loc.cpu().numpy().T
    R = np.triu(W[:res.achieved, :])
    assert np.abs(R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()
    assert [res.counters.trailing_passes, res.counters.blas3_volume] == \
        [ref.counters.trailing_passes, ref.counters.blas3_volume]
    single = G.rqrcp(A, k, b=b, p=p, seed=11, omega=om)
    assert np.array_equal(single.perm, res.perm)


@pytest.mark.parametrize("kind", ["short_panel", "lowrank"])
def test_block_cyclic_gpu_lazy_exits(nccl1, kind):
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
    A_loc = torch.from_numpy(np.ascontiguousarray(A.T)).to(dev)
    res = rqrcp_block_cyclic(A_loc, m, n, n, b, p, 13, TorchComm(), GpuOps(dev), omega=om)
    ref = O.rqrcp(A, n, b=b, p=p, seed=13)
    assert res.achieved == ref.achieved_rank
    assert [res.counters.trailing_passes, res.counters.blas3_volume] == \
        [ref.counters.trailing_passes, ref.counters.blas3_volume]
    W = A_loc.cpu().numpy().T
    R = np.triu(W[:res.achieved, :])
    d = np.nonzero(res.perm != ref.perm)[0]
    if d.size:  # documented near-tie: pivots among columns already at the noise floor
        j, dr = int(d[0]), np.abs(ref.r_diag)
        assert j >= res.achieved or dr[j] <= 1e-10 * dr[0]
        assert np.abs(np.abs(np.diag(R))[:j] - dr[:j]).max() <= 1e-10 * dr[0]
        return
    assert np.abs(R - ref.R).max() <= 1e-10 * np.abs(ref.R).max()

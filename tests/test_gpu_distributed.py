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

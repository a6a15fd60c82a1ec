"""Multi-GPU code path on one GPU.  Only one B200 is available
to this build, and ranks that wait on one another must not share a GPU
(B200_PROFILING.md), so the NCCL path is exercised with a ONE-rank
communicator: the per-step reduce -> ncclAllReduce (C2), the sketch
allreduce (C3), the LSQR pass allreduce (C4), the gathered-x buffer of the
CSR SpMV (C1) and the NCCL calls inside the captured basis graph all run, and
must reproduce the single-GPU path BITWISE (same fixed-order sums; a 1-rank
allreduce is an identity).  The halo exchange and the multi-rank data
movement are covered on CPU by tests/test_dist_cpu.py."""
import os
import socket

import numpy as np
import pytest

import fab_problems as fp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    from paper_2212_12758_b200 import dist as fdist
    c = fdist.Comm(device=0)
    yield c
    c.close()
    dist.destroy_process_group()


def _solve(p, comm, csr=False, mode="blendenpik", fused=True, square=False):
    import torch
    import paper_2212_12758_b200 as fab
    from paper_2212_12758_b200 import dist as fdist
    op = fdist.local_operator(p, 0, p.n, csr=csr) if comm is not None else fab.Operator.from_problem(p, csr=csr)
    sv = fab.Solver(op, torch.as_tensor(p.b).cuda(), m_max=p.m, k_max=p.k, s_max=p.s, comm=comm, square=square)
    sv._op = op
    if fused:
        sv.sketch(p.s, p.sketch_seed)
    sv.basis(p.m, p.k)
    if not fused:
        sv.sketch(p.s, p.sketch_seed)
    sv.compress(mode, iters=40)
    y = sv.apply("sign" if square else p.f, 1.0 if square else p.alpha, p.sigma).cpu().numpy()
    out = dict(y=y, H=sv.get("H"), SV=sv.get("SV"), info=sv.info())
    sv.close()
    return out


@pytest.mark.parametrize("name,kw,csr", [
    ("c3", dict(g=32, m=40, s=80), False),
    ("c3", dict(g=24, m=30, s=60), True),
    ("c5", dict(n=5000, m=30, s=60), True),
])
def test_one_rank_nccl_path_is_bitwise_single_gpu(comm, name, kw, csr):
    p = fp.make(name, **kw)
    a = _solve(p, None, csr=csr)
    b = _solve(p, comm, csr=csr)
    assert np.array_equal(a["H"], b["H"])
    assert np.array_equal(a["SV"], b["SV"])
    assert np.array_equal(a["y"], b["y"])
    assert a["info"]["lsqr_iters"] == b["info"]["lsqr_iters"] == 40


@pytest.mark.parametrize("name,kw,csr", [
    ("e4", dict(n=5000, m=20, s=48), True),       # CSR: x and A x gathered
    ("e5", dict(g=16, m=20, s=48), False),       # stencil: halo of x and of A x
])
def test_one_rank_nccl_squared_operator(comm, name, kw, csr):
    """FAB_FLAG_SQUARE on the NCCL path (two C1 exchanges per step)."""
    p = fp.make(name, **kw)
    a = _solve(p, None, csr=csr, square=True)
    b = _solve(p, comm, csr=csr, square=True)
    assert np.array_equal(a["H"], b["H"]) and np.array_equal(a["y"], b["y"])


def test_one_rank_nccl_batched_sketch(comm):
    p = fp.make("c1", g=40, m=20, s=40)
    a = _solve(p, None, fused=False, mode="sketch_solve")
    b = _solve(p, comm, fused=False, mode="sketch_solve")
    assert np.array_equal(a["SV"], b["SV"]) and np.array_equal(a["y"], b["y"])


def test_p2p_mailboxes_carry_c2(comm, monkeypatch):
    """The per-step reduction (C2) goes through the NVLink mailboxes
    (fab_comm_p2p; with one rank the mailbox is this GPU's own): K1 posts,
    K3 collects, no ncclAllReduce in the step -- and the result is still
    bitwise the single-GPU one (test above) and the NCCL path's."""
    import torch
    from paper_2212_12758_b200 import dist as fdist
    assert comm.p2p
    p = fp.make("c3", g=32, m=40, s=80)
    a = _solve(p, comm)
    monkeypatch.setenv("FAB_P2P", "0")
    c2 = fdist.Comm(device=0)
    assert not c2.p2p
    b = _solve(p, c2)
    c2.close()
    assert np.array_equal(a["y"], b["y"]) and np.array_equal(a["H"], b["H"])
    torch.cuda.synchronize()


def test_partition_validation(comm):
    """A 1-rank communicator must own every row: fab_init refuses a block
    that does not tile [0, n) (EINVAL), and an unaligned block start."""
    import torch
    import paper_2212_12758_b200 as fab
    from paper_2212_12758_b200 import FabError
    p = fp.make("c3", g=16, m=10, s=20)
    op = fab.Operator.stencil(p.dims, p.coeffs, rows=(0, p.n - 256))
    with pytest.raises(FabError):
        fab.Solver(op, torch.as_tensor(p.b[: p.n - 256]).cuda(), 10, 4, 20, comm=comm)
    op = fab.Operator.stencil(p.dims, p.coeffs, rows=(16, p.n))
    with pytest.raises(FabError):
        fab.Solver(op, torch.as_tensor(p.b[16:]).cuda(), 10, 4, 20, comm=comm)

"""Multi-GPU path, CPU side: the product's partition plans
(paper_2212_12758_b200.dist) and a world-size-2 `gloo` run of the
row-partitioned decomposition (tests/dist_model.py: halo exchange, one
allreduce per Krylov step, tile-aligned SRHT partials across non-aligned row
blocks, allreduced LSQR scalars) against the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import fab_problems as fp
from paper_2212_12758_b200 import dist as fdist


def test_stencil_blocks_are_slabs():
    cuts = fdist.stencil_blocks((256, 256, 256), 8)
    assert list(np.diff(cuts)) == [32 * 65536] * 8            # 32 planes each (c3, P = 8)
    cuts = fdist.stencil_blocks((64, 64, 10), 4)              # 10 planes over 4: 3,3,2,2
    assert list(np.diff(cuts) // 4096) == [3, 3, 2, 2]
    with pytest.raises(ValueError):
        fdist.stencil_blocks((64, 64, 3), 4)                  # fewer planes than ranks


def test_stencil_blocks_unaligned_planes_fall_back_to_rows():
    dims = (100, 100)                                         # 2D, line = 100 rows (not 32-aligned)
    cuts = fdist.stencil_blocks(dims, 3)
    assert cuts[0] == 0 and cuts[-1] == 10000
    assert all(c % 32 == 0 for c in cuts[:-1])
    assert np.diff(cuts).min() >= fdist.stencil_halo(dims)


def test_csr_blocks_balance_nnz():
    p = fp.make("c4", n=1 << 14, m=10, s=20)
    ip, _, _ = p.csr()
    cuts = fdist.csr_blocks(ip, 4)
    assert cuts[0] == 0 and cuts[-1] == p.n and all(c % 32 == 0 for c in cuts[:-1])
    nnz = np.diff(ip[cuts])
    assert nnz.max() <= 1.1 * nnz.mean()                      # hubs at low ids: rows are NOT equal
    rows = np.diff(cuts)
    assert rows.max() > 1.5 * rows.min()


def test_local_csr_rows_keep_global_columns():
    p = fp.make("c5", n=4096, m=5, s=10)
    ip, ix, dv = p.csr()
    lip, lix, ldv = fdist.local_csr(ip, ix, dv, 1024, 2048)
    assert lip[0] == 0 and len(lip) == 1025
    A = p.scipy()
    import scipy.sparse as sp
    Al = sp.csr_matrix((ldv, lix, lip), shape=(1024, p.n))
    assert (abs(Al - A[1024:2048]) > 0).nnz == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, P, port, case, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        import dist_model
        name, kw = case[:2]
        square = len(case) > 2 and case[2] == "square"
        p = fp.make(name, **kw)
        A = p.scipy()
        if p.kind == "stencil":
            cuts = fdist.stencil_blocks(p.dims, P)
            hal = fdist.stencil_halo(p.dims)
        else:
            cuts = fdist.csr_blocks(p.csr()[0], P)
            hal = None                                        # CSR: x gathered (all-gather-v)
        f = "invsqrt" if square else p.f
        fm, H, SV, y = dist_model.rank_solve(rank, P, A, p.b, cuts, hal, p.m, p.k, p.s, p.sketch_seed,
                                             f, p.alpha, p.sigma, 40, square=square)
        q.put((rank, cuts[rank], fm, H, SV, y))
    except BaseException as e:  # report instead of leaving the parent waiting
        q.put((rank, None, repr(e), None, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    ("c3", dict(g=16, m=30, k=4, s=60)),       # 3D stencil, 4096-row slabs of 16 planes -> halo = 1 plane
    ("c1", dict(g=64, m=24, k=2, s=48)),       # 2D, 64-row lines; blocks not tile aligned
    ("c5", dict(n=6000, m=20, k=2, s=40)),     # CSR, ragged n, row blocks cut mid-tile
    # squared operator (sign(A) b = (A^2)^{-1/2} (A b), l.406): two C1 exchanges per step
    ("e4", dict(n=6000, m=20, k=2, s=40), "square"),     # CSR: x and A x gathered
    ("e5", dict(g=16, m=20, k=2, s=40), "square"),       # stencil: halo of x and of A x
])
def test_row_partitioned_solve_matches_oracle_gloo(case):
    from oracle import fab as ofab
    P = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, case, q)) for r in range(P)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(P)], key=lambda t: t[0])
    for r in res:
        assert r[1] is not None, r[2]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    name, kw = case[:2]
    p = fp.make(name, **kw)
    if len(case) > 2:
        ref = ofab.sign(p.scipy(), p.b, p.m, p.k, p.s, p.sketch_seed, mode="blendenpik", lsqr_iters=40)
    else:
        ref = ofab.solve(p.scipy(), p.b, p.m, p.k, p.s, p.sketch_seed, mode="blendenpik", f=p.f,
                         alpha=p.alpha, sigma=p.sigma, lsqr_iters=40, variant="cgs")
    fm = np.concatenate([r[2] for r in res])
    assert res[1][1] % 4096 != 0 or name in ("c3", "e5")      # a block boundary inside a sketch tile
    for r in res:                                             # replicated quantities agree
        assert np.array_equal(r[3], res[0][3]) and np.array_equal(r[4], res[0][4])
    H, SV = res[0][3], res[0][4]
    assert np.abs(H - ref["H"]).max() <= 1e-12 * np.abs(ref["H"]).max()
    assert np.abs(SV - ref["SV"]).max() <= 1e-13 * max(1.0, np.abs(ref["SV"]).max())
    rel = np.linalg.norm(fm - ref["f_m"]) / np.linalg.norm(ref["f_m"])
    assert rel <= 1e-10, rel

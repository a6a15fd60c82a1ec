"""Small solves that run every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck; SURVEY §5 "race detection"):

    compute-sanitizer --tool racecheck python profiles/sanitize_driver.py

K1 (stencil vector path and CSR), K3 with the fused sketch (bulk-copy ring,
mbarriers), K5 (both kernels), the K6 TMA pipeline in the graph-resident and
host-driven LSQR loops, the Blendenpik preconditioner sketch, the sketch QR
and triangular inverse, Denman-Beavers with the cluster Gauss-Jordan
inverse (DSMEM), Pade exp, the final combination, Algorithm 1 and Arnoldi's
tall GEMVs, and a two-rank loopback solve (halo on a side stream).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402
from paper_2212_12758_b200 import dist as fdist  # noqa: E402


def solve(p, profile=False, csr=False):
    sv = fab.Solver(fab.Operator.from_problem(p, csr=csr), torch.as_tensor(p.b).cuda(), p.m, p.k, 2 * p.s,
                    profile=profile)
    sv.sketch(p.s, p.sketch_seed)
    sv.basis(p.m, p.k)                                   # K1 + K3 (fused sketch)
    sv.compress("blendenpik", tol=1e-6)                  # QR, R^-1, K6 loop
    y = sv.apply(p.f, p.alpha, p.sigma)                  # dense f + K7
    sv.compress("blendenpik", iters=10, precond_s=2 * p.s, precond_seed=5)   # K5 with Theta'
    sv.apply(p.f, p.alpha, p.sigma)
    for k5 in ("1", "2"):                                # API order: K5 direct / tile groups
        os.environ["FAB_SKETCH_K5"] = k5
        sv.basis(p.m, p.k)
        sv.sketch(p.s, p.sketch_seed + 1)
        sv.compress("sketch_solve")
    sv.sketch(p.s, p.sketch_seed)
    sv.basis_sgs(min(p.m, 20))                           # Algorithm 1
    sv.basis_arnoldi(min(p.m, 20))                       # CGS2
    torch.cuda.synchronize()
    sv.close()
    return y


torch.cuda.set_device(0)
solve(fp.make("c3", g=32, m=40, s=80))                   # sqrt: Denman-Beavers, cluster Gauss-Jordan
solve(fp.make("c3", g=32, m=40, s=80), profile=True)     # host-driven LSQR loop
solve(fp.make("c5", n=20000, m=30, s=60), csr=True)      # CSR K1, invsqrt
solve(fp.make("c1"))                                     # exp: Pade
p = fp.make("c3", g=32, m=30, s=60)
cuts = fdist.stencil_blocks(p.dims, 2)
grp = fdist.LoopbackGroup(2, 0)


def rank(r, comm, st):
    op = fdist.local_operator(p, int(cuts[r]), int(cuts[r + 1]))
    b = torch.as_tensor(np.ascontiguousarray(p.b[cuts[r]:cuts[r + 1]])).cuda()
    sv = fab.Solver(op, b, p.m, p.k, p.s, stream=st, comm=comm)
    sv.sketch(p.s, p.sketch_seed)
    sv.basis(p.m, p.k)
    sv.compress("blendenpik", iters=10)
    sv.apply(p.f, p.alpha, p.sigma)
    st.synchronize()
    sv.close()


grp.run(rank)
grp.close()
print("sanitize driver done")

"""The CSR K1 plan cache (csr.cu: row blocks, uniform-value detection, the
column-blocked copy) is shared by the contexts of one operator.  A context
created on arrays at the SAME device addresses but with different contents
(an address the caching allocator hands to a new operator) must get its own
plan: the cache key carries a content fingerprint."""
import numpy as np
import pytest

import fab_problems as fp
from oracle import fab as ofab

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def test_plan_not_reused_across_contents_at_same_address():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    import scipy.sparse as sp
    import paper_2212_12758_b200 as fab
    p = fp.make("c4", n=1 << 14, m=20, s=40)          # 0/1 adjacency / lambda: uniform values
    ip, ix, dv = p.csr()
    assert np.all(dv == dv[0])
    op = fab.Operator.csr(ip, ix, dv)
    b = torch.as_tensor(p.b).cuda()
    sv1 = fab.Solver(op, b, p.m, p.k, p.s)             # plan: uniform (values dropped)
    sv1.sketch(p.s, p.sketch_seed)
    sv1.basis(p.m, p.k)
    sv1.compress("sketch_solve")
    y1 = sv1.apply(p.f, p.alpha, p.sigma).cpu().numpy()
    assert rel(y1, ofab.solve(p.scipy(), p.b, p.m, p.k, p.s, p.sketch_seed, mode="sketch_solve", f=p.f,
                              alpha=p.alpha, sigma=p.sigma)["f_m"]) <= 1e-10
    # new contents at the same addresses (sv1 still alive, holding the plan)
    dv2 = dv * (1.0 + 0.5 * np.random.default_rng(3).random(len(dv)))
    vals = op._keep[2]
    vals.copy_(torch.as_tensor(dv2))
    torch.cuda.synchronize()
    sv2 = fab.Solver(op, b, p.m, p.k, p.s)
    sv2.sketch(p.s, p.sketch_seed)
    sv2.basis(p.m, p.k)
    sv2.compress("sketch_solve")
    y2 = sv2.apply(p.f, p.alpha, p.sigma).cpu().numpy()
    A2 = sp.csr_matrix((dv2, ix, ip), shape=(p.n, p.n))
    ref2 = ofab.solve(A2, p.b, p.m, p.k, p.s, p.sketch_seed, mode="sketch_solve", f=p.f, alpha=p.alpha,
                      sigma=p.sigma)
    assert rel(y2, ref2["f_m"]) <= 1e-10
    sv1.close()
    sv2.close()

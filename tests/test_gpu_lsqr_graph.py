"""The graph-resident LSQR loop (one CUDA graph: init pass, then a
conditional WHILE node whose body is one iteration; k_lsqr_step sets the
condition on the device, so MATLAB lsqr's tolerance test (PAPER.md l.359,
reading G-14) needs no host round trip) against the host-driven loop
(FAB_FLAG_PROFILE, or FAB_LSQR_GRAPH=0): the same kernels in the same order,
so the iterate, the iteration count and f_m must be bitwise equal, in both
the tolerance and the fixed-L (parity) mode, at every pipe instantiation."""
import numpy as np
import pytest

import fab_problems as fp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def solve(p, profile, **kw):
    import torch
    import paper_2212_12758_b200 as fab
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s, profile=profile)
    out = []
    for _ in range(2):                 # the second call replays the cached graph
        sv.sketch(p.s, p.sketch_seed)
        sv.basis(p.m, p.k)
        sv.compress("blendenpik", **kw)
        y = sv.apply(p.f, p.alpha, p.sigma).cpu().numpy()
        out.append((y, sv.get("y"), sv.info()))
    sv.close()
    return out


@pytest.mark.parametrize("name,kw", [
    ("c1", {}),
    ("c2", dict(g=300, m=100, s=200)),
    ("c5", dict(n=1 << 16, m=200, s=400)),
    ("c5", dict(n=1 << 15, m=300, s=600)),
])
@pytest.mark.parametrize("mode", [dict(tol=1e-6), dict(iters=40), dict(tol=1e-6, maxit=7)])
def test_graph_loop_bitwise_equals_host_loop(name, kw, mode):
    p = fp.make(name, **kw)
    ref = solve(p, True, **mode)       # FAB_FLAG_PROFILE: host-driven loop, CUDA events per pass
    got = solve(p, False, **mode)      # graph-resident loop
    for (y0, ls0, i0), (y1, ls1, i1) in zip(ref, got):
        assert i1["lsqr_iters"] == i0["lsqr_iters"]
        assert i1["lsqr_converged"] == i0["lsqr_converged"]
        assert np.array_equal(ls1, ls0) and np.array_equal(y1, y0)
        assert i1["lsqr_rnorm"] == i0["lsqr_rnorm"]
    if "maxit" in mode:                # the cap ends the while loop too
        assert got[0][2]["lsqr_iters"] == 7
    if "iters" in mode:
        assert got[0][2]["lsqr_iters"] == 40

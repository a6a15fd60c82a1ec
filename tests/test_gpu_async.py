"""FAB_FLAG_ASYNC (only fab_apply synchronizes): fab_basis and
fab_compress only enqueue; their status is resolved at fab_apply.  The
result must be bitwise the synchronous one -- including after a lucky
breakdown (reading G-5), where the compression enqueued for
m columns is redone on the m_eff columns at the resolution."""
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


def run(p, asynchronous, mode, **kw):
    import torch
    import paper_2212_12758_b200 as fab
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s,
                    asynchronous=asynchronous)
    out = []
    for _ in range(2):
        if mode != "none":
            sv.sketch(p.s, p.sketch_seed)
        st_b = sv.basis(p.m, p.k)
        st_c = sv.compress(mode, **kw)
        y = sv.apply(p.f, p.alpha, p.sigma).cpu().numpy()
        out.append((y, sv.get("y"), sv.info(), st_b, st_c, sv.status["apply"]))
    sv.close()
    return out


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c3", dict(g=40, m=60, s=120)),
                                     ("c5", dict(n=1 << 15, m=200, s=400))])
@pytest.mark.parametrize("mode,opts", [("blendenpik", dict(tol=1e-6)), ("blendenpik", dict(iters=40)),
                                       ("sketch_solve", {}), ("none", {})])
def test_async_bitwise_equals_sync(name, kw, mode, opts):
    p = fp.make(name, **kw)
    ref = run(p, False, mode, **opts)
    got = run(p, True, mode, **opts)
    for (y0, l0, i0, *_), (y1, l1, i1, b1, c1, a1) in zip(ref, got):
        assert np.array_equal(y1, y0) and np.array_equal(l1, l0)
        for key in ("lsqr_iters", "lsqr_converged", "m_eff", "breakdown", "cond_R", "gamma_b"):
            assert i1[key] == i0[key], key
        assert b1 == 0 and c1 == 0 and a1 >= 0
        assert i1["ms_basis"] > 0


def test_async_breakdown_redoes_compression():
    import scipy.sparse as sp
    import torch
    import paper_2212_12758_b200 as fab
    vals = np.repeat([-0.5, -1.0, -2.0, -3.0, -4.0], 40)
    A = sp.diags(vals).tocsr()
    b = np.random.default_rng(0).standard_normal(len(vals))
    for mode in ("blendenpik", "sketch_solve", "none"):
        sv = fab.Solver(fab.Operator.csr(A.indptr, A.indices, A.data), torch.as_tensor(b).cuda(), 10, 2, 20,
                        asynchronous=True)
        sv.sketch(20, 1)
        assert sv.basis(10, 2) == 0                 # enqueued: the breakdown is not known yet
        assert sv.compress(mode, iters=40) == 0
        y = sv.apply("exp", 1.0, 0.0).cpu().numpy()
        assert sv.status["apply"] == 1              # FAB_BREAKDOWN, reported by the resolving call
        inf = sv.info()
        assert inf["m_eff"] == 5 and inf["breakdown"] == 1
        assert np.linalg.norm(y - np.exp(vals) * b) <= 1e-12 * np.linalg.norm(b)
        sv.close()

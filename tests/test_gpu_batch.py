"""Multi-RHS (fab_basis_batch): p contexts of one operator
built in one graph, the CSR entries read once per Krylov step for all of
them.  Each context must end in exactly the state of its own fab_basis
(bitwise: same kernels, grids and per-vector reduction order), and f_m must
match the oracle at BASELINE's 1e-10."""
import numpy as np
import pytest

import fab_problems as fp
from oracle import fab as ofab

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def rhs(p, i):
    """b_0 = the problem's b, others seeded N(0,1) (the multi-RHS inputs)."""
    return p.b if i == 0 else np.random.default_rng(7000 + i).standard_normal(p.n)


def solvers(p, op, nb, square=False, fused=True):
    import torch
    import paper_2212_12758_b200 as fab
    out = []
    for i in range(nb):
        sv = fab.Solver(op, torch.as_tensor(rhs(p, i)).cuda(), p.m, p.k, p.s, square=square)
        if fused:
            sv.sketch(p.s, p.sketch_seed)
        out.append(sv)
    return out


@pytest.mark.parametrize("name,kw,nb,colblock,batchblock,square", [
    ("c5", dict(n=5001, m=15, s=40), 3, None, None, False),
    ("c4", dict(n=1 << 14, m=20, s=50), 4, None, None, False),     # hub rows (long-row path)
    ("c5", dict(n=5001, m=15, s=40), 2, "1000", None, False),      # column-blocked passes
    ("e4", dict(n=5001, m=15, s=40), 3, None, None, True),         # squared operator: K0 and K1 batched
    ("c1", dict(m=30), 3, None, None, False),                       # stencil: per-context K1
    # a column-blocked plan built for the batch only (the contexts' own plan is
    # one pass): the c4 p = 4 layout at full size, where the interleaved copy
    # exceeds L2; S = 4 (256-bit gathers) at p = 4 and p = 3, S = 2 at p = 2
    ("c4", dict(n=1 << 14, m=20, s=50), 4, None, "3001", False),
    ("c4", dict(n=1 << 14, m=20, s=50), 3, None, "5000", False),
    ("c5", dict(n=5001, m=15, s=40), 2, None, "1700", False),
])
def test_batch_equals_single_and_oracle(name, kw, nb, colblock, batchblock, square, monkeypatch):
    import paper_2212_12758_b200 as fab
    if colblock:
        monkeypatch.setenv("FAB_CSR_COLBLOCK", colblock)
    p = fp.make(name, **kw)
    op = fab.Operator.from_problem(p)
    f = "sign" if square else p.f
    alpha = 1.0 if square else p.alpha
    batch = solvers(p, op, nb, square)
    if batchblock:
        monkeypatch.setenv("FAB_BATCH_COLBLOCK", batchblock)
    fab.basis_batch(batch, p.m, p.k)
    if batchblock:   # the single solves use the batch's plan width, so bitwise equality is defined
        monkeypatch.setenv("FAB_CSR_COLBLOCK", batchblock)
    single = solvers(p, op, nb, square)
    for sv in single:
        sv.basis(p.m, p.k)
    A = p.scipy()
    for i in range(nb):
        a, b = batch[i], single[i]
        if batchblock is None:
            assert np.array_equal(a.get("H"), b.get("H"))                   # bitwise
            assert np.array_equal(a.get("SV"), b.get("SV"))
            assert np.array_equal(a.get("beta"), b.get("beta"))
        else:
            # same plan, but K1's grid follows each context's own plan (the
            # dot partials are summed over another CTA count): rounding only
            assert rel(a.get("H"), b.get("H")) <= 1e-13
            assert rel(a.get("SV"), b.get("SV")) <= 1e-13
        a.compress("blendenpik", iters=40)
        b.compress("blendenpik", iters=40)
        ya = a.apply(f, alpha, p.sigma).cpu().numpy()
        yb = b.apply(f, alpha, p.sigma).cpu().numpy()
        if batchblock is None:
            assert np.array_equal(ya, yb)
        if square:
            ref = ofab.sign(A, rhs(p, i), p.m, p.k, p.s, p.sketch_seed, mode="blendenpik", lsqr_iters=40,
                            keep=False)
        else:
            ref = ofab.solve(A, rhs(p, i), p.m, p.k, p.s, p.sketch_seed, mode="blendenpik", f=p.f,
                             alpha=p.alpha, sigma=p.sigma, lsqr_iters=40, keep=False)
        assert rel(ya, ref["f_m"]) <= 1e-10, (i, rel(ya, ref["f_m"]))
    for sv in batch + single:
        sv.close()


def test_batch_unfused_and_repeat():
    """No sketch (Algorithm 5), then the cached graph again with new b."""
    import paper_2212_12758_b200 as fab
    p = fp.make("c5", n=4000, m=12, s=30)
    op = fab.Operator.from_problem(p)
    batch = solvers(p, op, 2, fused=False)
    for rep in range(2):
        if rep:
            for i, sv in enumerate(batch):
                sv.set_b(rhs(p, i + 5))
        fab.basis_batch(batch, p.m, p.k)
        for i, sv in enumerate(batch):
            sv.compress("none")
            y = sv.apply(p.f, p.alpha, p.sigma).cpu().numpy()
            b = rhs(p, i + 5 if rep else i)
            ref = ofab.solve(p.scipy(), b, p.m, p.k, p.s, p.sketch_seed, mode="none", f=p.f, alpha=p.alpha,
                             keep=False)
            assert rel(y, ref["f_m"]) <= 1e-10


def test_batch_breakdown_in_one_context():
    """A diagonal A and one b that is an eigenvector: that context breaks down
    at step 1, the others run to m; every result is exact or the oracle's."""
    import scipy.sparse as sp
    import torch
    import paper_2212_12758_b200 as fab
    vals = np.repeat([-0.5, -1.0, -2.0, -3.0, -4.0, -5.0], 50)
    A = sp.diags(vals).tocsr()
    n = len(vals)
    op = fab.Operator.csr(A.indptr, A.indices, A.data)
    e = np.zeros(n)
    e[3] = 1.0
    bs = [np.random.default_rng(1).standard_normal(n), e]
    svs = [fab.Solver(op, torch.as_tensor(b).cuda(), 8, 2, 0) for b in bs]
    st = fab.basis_batch(svs, 8, 2)
    assert st == 1                                            # FAB_BREAKDOWN (warning)
    assert [sv.info()["m_eff"] for sv in svs] == [6, 1]
    for sv, b in zip(svs, bs):
        sv.compress("none")
        y = sv.apply("exp").cpu().numpy()
        assert rel(y, np.exp(vals) * b) <= 1e-12


def test_batch_rejects_mismatched_contexts():
    import torch
    import paper_2212_12758_b200 as fab
    from paper_2212_12758_b200 import FabError
    p = fp.make("c5", n=3000, m=10, s=30)
    q = fp.make("c5", n=3000, m=10, s=30)
    opa, opb = fab.Operator.from_problem(p), fab.Operator.from_problem(q)   # distinct arrays
    a = fab.Solver(opa, torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
    b = fab.Solver(opb, torch.as_tensor(q.b).cuda(), q.m, q.k, q.s)
    with pytest.raises(FabError):
        fab.basis_batch([a, b], p.m, p.k)
    with pytest.raises(FabError):
        fab.basis_batch([a, a], p.m, p.k)
    with pytest.raises(FabError):
        fab.basis_batch([a] * 5, p.m, p.k)

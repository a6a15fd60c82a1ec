"""Parity at full size for the CSR path and the paper's 3D Laplacian:

c5 (BASELINE.json: n = 2^25 random sparse, 16 + 1 entries per row, m = 300,
k = 2, s = 600, f = invsqrt of -A) in the launch configuration
profiles/bench_configs.py times -- the column-blocked K1 (x = 268 MB exceeds
the L2 budget, so fab_init regroups the entries into column blocks) -- on
sampled outputs the oracle computes one by one and on properties that hold
at any size:
  * sampled rows / sign bits of Theta bit-exact at N = 2^25;
  * entries of Theta V = the oracle's one-entry definition on the GPU basis;
  * the Arnoldi-like relation A V_m = V_{m+1} H_m on sampled rows (each row
    of A from the CSR, its 17 columns scattered over all column blocks);
  * window orthogonality of the last columns; sketch-and-solve y = the
    oracle's QR solve of the GPU sketch; f_m rows = gamma V c; the three
    modes agree (c5 converges like 5^-m).

e5 (3D Laplacian N = 80, n = 512,000, invsqrt,
s = floor(1.05 m)) at m = 300: f_m against the exact A^{-1/2} b (DST-I closed
form) within the method's own error, and equal to the oracle's Algorithm 4.
"""
import numpy as np
import pytest

import fab_problems as fp
from oracle import fab as ofab
from oracle import lsq as olsq
from oracle import rng as orng
from oracle.srht import SRHT

pytestmark = pytest.mark.gpu


def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.fixture(scope="module")
def c5():
    _cuda()
    import torch
    import paper_2212_12758_b200 as fab
    p = fp.make("c5")
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
    out = {}
    for mode in ("sketch_solve", "none", "blendenpik"):
        sv.sketch(p.s, p.sketch_seed)
        sv.basis(p.m, p.k)
        sv.compress(mode, tol=1e-6)
        out[mode] = sv.apply(p.f, p.alpha, p.sigma).cpu().numpy()
        if mode == "sketch_solve":
            out["y_ss"] = sv.get("y")
    yield p, sv, out
    sv.close()


def test_c5_rows_and_signs_bit_exact(c5):
    p, sv, _ = c5
    N = 1 << 25
    assert np.array_equal(sv.get("rows"), orng.rows(p.sketch_seed, N, p.s))
    bits = np.unpackbits(sv.get("signs").view(np.uint8), bitorder="little")[:N]
    assert np.array_equal(bits, (orng.signs(p.sketch_seed, N) < 0).astype(np.uint8))


def test_c5_sketch_entries(c5):
    p, sv, _ = c5
    SV = sv.get("SV")
    th = SRHT(p.n, p.s, p.sketch_seed)
    rng = np.random.default_rng(5)
    for j in (0, 1, 150, 300):
        v = sv.column(j)
        for q in rng.choice(p.s, 2, replace=False):
            ref = th.row_entry(int(th.rows[q]), v)
            assert abs(SV[q, j] - ref) <= 1e-13 * np.abs(SV[:, j]).max(), (j, q)


def test_c5_arnoldi_relation_and_window(c5):
    p, sv, _ = c5
    ip, ix, dv = p.csr()
    H = sv.get("H")
    rng = np.random.default_rng(6)
    rows = np.sort(rng.choice(p.n, 24, replace=False))
    rows[0], rows[-1] = 0, p.n - 1
    worst = 0.0
    for r in rows:
        cols, vals = ix[ip[r]:ip[r + 1]].astype(np.int64), dv[ip[r]:ip[r + 1]]
        Vn = sv.vrows(cols)
        Vr = sv.vrows([r])[0]
        lhs = vals @ Vn[:, : p.m]
        rhs = Vr @ H
        worst = max(worst, np.abs(lhs - rhs).max() / (p.norm_inf * max(1e-300, np.abs(Vn).max())))
    assert worst <= 1e-12, worst
    cols = [sv.column(j) for j in range(p.m - p.k, p.m + 1)]
    for a in range(len(cols)):
        assert abs(np.linalg.norm(cols[a]) - 1.0) <= 1e-13
        for b in range(a):
            assert abs(cols[a] @ cols[b]) <= 1e-12


def test_c5_sketch_and_solve_y_and_combination(c5):
    p, sv, out = c5
    SV = sv.get("SV")
    y, _ = olsq.sketch_and_solve(SV[:, : p.m], SV[:, p.m])
    assert np.linalg.norm(out["y_ss"] - y) <= 1e-10 * np.linalg.norm(y)
    info = sv.info()
    c = sv.get("fc")
    rows = np.random.default_rng(7).choice(p.n, 64, replace=False)
    ref = info["gamma_b"] * (sv.vrows(rows)[:, : p.m] @ c)
    assert np.abs(out["blendenpik"][rows] - ref).max() <= 1e-13 * np.abs(out["blendenpik"]).max()


def test_c5_modes_agree(c5):
    _, _, out = c5
    ref = out["blendenpik"]
    assert np.isfinite(ref).all()
    for mode in ("sketch_solve", "none"):
        assert np.linalg.norm(out[mode] - ref) <= 1e-10 * np.linalg.norm(ref), mode


def test_e5_fullsize_against_closed_form():
    _cuda()
    import torch
    import paper_2212_12758_b200 as fab
    from test_oracle_paper_workloads import dst_invsqrt
    p = fp.make("e5", m=300)                              # N = 80, s = 315
    exact = dst_invsqrt(80, p.b)
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
    sv.sketch(p.s, p.sketch_seed)
    sv.basis(p.m, p.k)
    sv.compress("none")
    y = sv.apply("invsqrt").cpu().numpy()
    sv.close()
    ref = ofab.solve(p.scipy(), p.b, p.m, p.k, p.s, p.sketch_seed, mode="none", f="invsqrt", keep=False)
    err_gpu = np.linalg.norm(y - exact) / np.linalg.norm(exact)
    err_orc = np.linalg.norm(ref["f_m"] - exact) / np.linalg.norm(exact)
    assert np.linalg.norm(y - ref["f_m"]) <= 1e-10 * np.linalg.norm(ref["f_m"])
    assert err_gpu <= 2e-9 and abs(err_gpu - err_orc) <= 1e-10, (err_gpu, err_orc)

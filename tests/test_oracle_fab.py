"""End-to-end pins for oracle/fab.py against what the paper and the
mathematics fix (Lemma 1 l.151-166, Eq. (6) l.167-171, §3.2, §3.3,
polynomial exactness l.329-330, exact reference l.358)."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

import fab_problems as fp
from oracle import fab, krylov

GOLD = os.path.join(os.path.dirname(__file__), "golden")
MODES = ("blendenpik", "sketch_solve", "none")


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_diagonal_exact_with_breakdown():
    # diagonal A with d <= m distinct eigenvalues: breakdown at step d+1 and
    # f_m is exact (invariant subspace)
    vals = np.repeat([-0.5, -1.0, -2.0, -3.0, -4.0], 40)
    A = sp.diags(vals).tocsr()
    b = np.random.default_rng(0).standard_normal(200)
    for mode in MODES:
        out = fab.solve(A, b, m=10, k=2, s=20, seed=1, mode=mode, f="exp")
        assert out["breakdown"] and out["m_eff"] == 5
        assert rel(out["f_m"], np.exp(vals) * b) <= 1e-12


def test_diagonal_exact_converged():
    vals = np.linspace(1.0, 2.0, 300)
    A = sp.diags(vals).tocsr()
    b = np.random.default_rng(1).standard_normal(300)
    for f, ref in [("exp", np.exp(-vals) * b), ("sqrt", np.sqrt(vals) * b),
                   ("invsqrt", b / np.sqrt(vals))]:
        alpha = -1.0 if f == "exp" else 1.0
        for mode in MODES:
            out = fab.solve(A, b, m=20, k=2, s=40, seed=2, mode=mode, f=f, alpha=alpha,
                            lsqr_iters=40)
            assert rel(out["f_m"], ref) <= 1e-10, (f, mode)


@pytest.mark.parametrize("mode", MODES)
def test_dense_reference_nonsymmetric(mode):
    # c5-type operator (spectrum of -A in a disk around 5): invsqrt(-A) b
    p = fp.make("c5", n=400, m=30, k=2, s=60)
    A, b = p.scipy(), p.b
    ref = fab.dense(A, b, "invsqrt", alpha=-1.0)
    out = fab.solve(A, b, 30, 2, 60, 7, mode=mode, f="invsqrt", alpha=-1.0, lsqr_iters=40)
    assert rel(out["f_m"], ref) <= 1e-10


@pytest.mark.parametrize("mode", MODES)
def test_dense_reference_graph_exp(mode):
    p = fp.make("c4", n=400, m=25, k=2, s=50)
    A, b = p.scipy(), p.b
    ref = fab.dense(A, b, "exp", alpha=1.0)
    out = fab.solve(A, b, 25, 2, 50, 9, mode=mode, f="exp", lsqr_iters=40)
    assert rel(out["f_m"], ref) <= 1e-10


@pytest.mark.parametrize("mode", MODES)
def test_polynomial_exactness(mode):
    # l.329-330: exact for every polynomial of degree <= m-1, all algorithms
    p = fp.make("c3", g=10, m=10, k=4, s=40)
    A, b = p.scipy(), p.b
    coef = np.random.default_rng(3).standard_normal(10)       # degree 9 = m-1
    alpha = 1.0 / p.norm_inf
    ref = fab.dense(A, b, "poly", alpha=alpha, poly=coef)
    out = fab.solve(A, b, 10, 4, 40, 5, mode=mode, f="poly", alpha=alpha, poly=coef,
                    lsqr_iters=60)
    assert rel(out["f_m"], ref) <= 1e-10


def test_polynomial_degree_m_is_not_exact():
    # degree m is outside the exactness class (l.329): error is visible
    p = fp.make("c3", g=10, m=6, k=4, s=40)
    A, b = p.scipy(), p.b
    coef = np.zeros(7)
    coef[6] = 1.0
    alpha = 1.0 / p.norm_inf
    ref = fab.dense(A, b, "poly", alpha=alpha, poly=coef)
    out = fab.solve(A, b, 6, 4, 40, 5, mode="none", f="poly", alpha=alpha, poly=coef)
    assert rel(out["f_m"], ref) > 1e-6


def test_lemma1_fom_equals_blendenpik_exact_ls():
    # Lemma 1 (l.151-166): V_m f(V_m^+ A V_m) V_m^+ b is basis independent ->
    # Alg 4 with an (essentially) exact LS solve equals Arnoldi FOM (Eq. 4)
    p = fp.make("c1", g=40, m=25, k=2, s=50)
    A, b = p.scipy(), p.b
    f_fom = fab.fom(A, b, 25, "exp", alpha=-1.0)
    out = fab.solve(A, b, 25, 2, 50, 11, mode="blendenpik", f="exp", alpha=-1.0,
                    lsqr_tol=1e-14, lsqr_maxit=200)
    assert rel(out["f_m"], f_fom) <= 1e-9


def test_alg5_equals_lanczos_fom_symmetric():
    # §3.2: Eq. (8) coincides with Eq. (4) when V_m is orthonormal: symmetric
    # A with k = 2 is Lanczos (l.104)
    n = 500
    A = sp.diags([-np.ones(n - 1), 2 + np.linspace(0, 1, n), -np.ones(n - 1)], [-1, 0, 1]).tocsr()
    b = np.random.default_rng(4).standard_normal(n)
    out = fab.solve(A, b, 20, 2, 40, 1, mode="none", f="exp", alpha=-1.0)
    assert rel(out["f_m"], fab.fom(A, b, 20, "exp", alpha=-1.0)) <= 1e-8


def test_eq6_last_column_structure():
    # Eq. (6): V_m^+ A V_m - H_m is zero outside its last column
    p = fp.make("c5", n=300, m=12, k=2, s=30)
    A, b = p.scipy(), p.b
    d = krylov.truncated_arnoldi(A, b, 12, 2)
    Vm = d["V"][:, :12]
    P = np.linalg.pinv(Vm) @ (A @ Vm)
    D = P - d["H"][:12, :12]
    assert np.abs(D[:, :11]).max() <= 1e-10 * np.abs(d["H"]).max()
    # ... and the last column is h_{m+1,m} V_m^+ v_{m+1}  (y of Eq. (7))
    y = np.linalg.lstsq(Vm, d["V"][:, 12], rcond=None)[0]
    assert np.allclose(D[:, 11], d["H"][12, 11] * y, atol=1e-10)
    # gamma_b contract: V_m (gamma e_1) = b
    assert rel(d["gamma"] * Vm[:, 0], b) <= 1e-15


def test_zero_matrix_and_eigenvector():
    # A = 0 -> f(0) b ; b eigenvector -> f(lambda) b at m = 1
    n = 64
    A = sp.csr_matrix((n, n))
    b = np.random.default_rng(5).standard_normal(n)
    out = fab.solve(A, b, 5, 2, 10, 1, mode="blendenpik", f="exp")
    assert out["m_eff"] == 1 and rel(out["f_m"], b) <= 1e-15
    out = fab.solve(A, b, 5, 2, 10, 1, mode="none", f="sqrt", sigma=4.0)
    assert rel(out["f_m"], 2 * b) <= 1e-15
    D = sp.diags(np.arange(1.0, n + 1)).tocsr()
    e = np.zeros(n)
    e[3] = 2.0
    out = fab.solve(D, e, 5, 2, 10, 1, mode="sketch_solve", f="sqrt")
    assert out["m_eff"] == 1 and rel(out["f_m"], 2.0 * e) <= 1e-15


def test_sfom_formula_equals_sketch_and_solve():
    # Remark 2 (l.249-251): sFOM Eq. (9) == Alg 2 + sketch-and-solve LS
    p = fp.make("c5", n=1000, m=20, k=2, s=40)
    A, b = p.scipy(), p.b
    for f, alpha in [("exp", 0.2), ("invsqrt", -1.0)]:
        a = fab.sfom(A, b, 20, 2, 40, 3, f=f, alpha=alpha)
        c = fab.solve(A, b, 20, 2, 40, 3, mode="sketch_solve", f=f, alpha=alpha)
        assert rel(c["f_m"], a) <= 1e-10


def test_sign_function_formula():
    # PAPER.md l.406 / S:491: sign(A) b = (A^2)^{-1/2} (A b); A = diag(2,-3), b = (1,1)
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["sign_diag"]
    A = np.array(g["A"])
    Ab = A @ np.array(g["b"])
    A2 = sp.csr_matrix(A @ A)
    out = fab.solve(A2, Ab, 2, 2, 2, 1, mode="none", f="invsqrt")
    assert np.allclose(out["f_m"], g["signAb"], atol=1e-12)


def test_modes_agree_when_converged_c2_small():
    # well-conditioned basis: every mode converges to the same f(A)b
    p = fp.make("c2", g=60, m=40, k=2, s=80)
    A, b = p.scipy(), p.b
    outs = [fab.solve(A, b, 40, 2, 80, 3002, mode=md, f="exp", alpha=-1e-3, lsqr_iters=40)
            for md in MODES]
    ref = fab.dense(A, b, "exp", alpha=-1e-3) if p.n <= 4000 else None
    for o in outs:
        assert rel(o["f_m"], ref) <= 1e-10


# ---- Algorithm 3 (Alg 1 basis + LSQR) -----------------
def test_alg3_exact_ls_equals_fom_lemma1():
    # Lemma 1 (l.151-166): with the exact least-squares y, Alg 3 = FOM Eq. (4)
    for name, kw in [("c1", dict(g=30, m=20, s=50)), ("c5", dict(n=2000, m=25, s=60))]:
        p = fp.make(name, **kw)
        A = p.scipy()
        r = fab.alg3(A, p.b, p.m, p.s, p.sketch_seed, f=p.f, alpha=p.alpha, sigma=p.sigma, lsqr_tol=1e-14)
        fo = fab.fom(A, p.b, p.m, f=p.f, alpha=p.alpha, sigma=p.sigma)
        assert np.linalg.norm(r["f_m"] - fo) <= 1e-9 * np.linalg.norm(fo), name


def test_alg3_polynomial_exactness():
    # l.329-330: polynomials of degree <= m-1 are reproduced exactly
    p = fp.make("c3", g=10, m=8, s=30)
    A = p.scipy()
    coef = np.random.default_rng(9).standard_normal(8)
    alpha = 1.0 / p.norm_inf
    r = fab.alg3(A, p.b, p.m, p.s, 5, f="poly", alpha=alpha, poly=coef, lsqr_tol=1e-14)
    ref = fab.dense(A, p.b, "poly", alpha=alpha, poly=coef)
    assert np.linalg.norm(r["f_m"] - ref) <= 1e-10 * np.linalg.norm(ref)


def test_alg3_converges_to_dense_exp():
    p = fp.make("c4", n=1 << 10, m=30, s=70)
    A = p.scipy()
    r = fab.alg3(A, p.b, p.m, p.s, p.sketch_seed, f=p.f, alpha=p.alpha, lsqr_tol=1e-14)
    ref = fab.dense(A, p.b, p.f, alpha=p.alpha)
    assert np.linalg.norm(r["f_m"] - ref) <= 1e-10 * np.linalg.norm(ref)


def test_whitened_alg4_on_graph_matches_dense_exp():
    # whitening makes the least-squares modes well posed on a Lanczos-like
    # problem (l.457-458); exp of the scaled graph is converged at m = 60
    p = fp.make("c4", n=1 << 12, m=60, s=130)
    A = p.scipy()
    ref = fab.dense(A, p.b, p.f, alpha=p.alpha)
    for mode in ("blendenpik", "sketch_solve", "none"):
        r = fab.solve_whitened(A, p.b, p.m, p.k, p.s, p.sketch_seed, mode=mode, f=p.f, alpha=p.alpha,
                               lsqr_iters=60)
        assert r["whitened_at"] > 0
        assert np.linalg.norm(r["f_m"] - ref) <= 1e-10 * np.linalg.norm(ref), mode


# ---- Blendenpik's own preconditioner sketch (reading G-12) --
def test_precond_same_sketch_is_default():
    """precond=(s, seed) is the basis sketch Theta itself: the same R, y, f_m."""
    p = fp.make("c2", g=60, m=30, s=60)
    a = fab.solve(p.scipy(), p.b, p.m, p.k, p.s, p.sketch_seed, mode="blendenpik", f=p.f, alpha=p.alpha,
                  lsqr_iters=20)
    b = fab.solve(p.scipy(), p.b, p.m, p.k, p.s, p.sketch_seed, mode="blendenpik", f=p.f, alpha=p.alpha,
                  lsqr_iters=20, precond=(p.s, p.sketch_seed))
    assert np.array_equal(a["R"], b["R"]) and np.array_equal(a["f_m"], b["f_m"])


def test_precond_isometric_sketch_makes_lsqr_one_step():
    """With s' = N the SRHT is an isometry (Theta'^T Theta' = I, G-9), so R is
    V_m's own R factor and V_m R^{-1} has orthonormal columns: LSQR on it
    terminates with the exact least-squares solution within two iterations
    (one distinct singular value), whatever the conditioning of V_m."""
    p = fp.make("c3", g=16, m=12, k=4, s=30)            # n = 4096 = N
    dec = krylov.truncated_arnoldi(p.scipy(), p.b, p.m, p.k, variant="cgs")
    from oracle.srht import SRHT
    SV = SRHT(p.n, p.s, p.sketch_seed).apply(dec["V"])
    y, C, R, info = fab.compress(dec, SV, "blendenpik", lsqr_tol=1e-12, precond=(p.n, 99))
    V = dec["V"]
    ref = np.linalg.lstsq(V[:, :p.m], V[:, p.m], rcond=None)[0]
    assert info["iters"] <= 2
    assert rel(y, ref) <= 1e-10
    Q = V[:, :p.m] @ np.linalg.inv(R)
    assert np.abs(Q.T @ Q - np.eye(p.m)).max() <= 1e-12


def test_precond_larger_sketch_fewer_iterations():
    """A larger preconditioner sketch gives a better-conditioned V_m R^{-1}
    (embedding distortion ~ sqrt(m/s')): fewer LSQR iterations to the MATLAB
    tolerance 1e-6 (l.359), and the same compression within that tolerance."""
    p = fp.make("c5", n=1 << 14, m=60, s=120)
    A = p.scipy()
    a = fab.solve(A, p.b, p.m, p.k, p.s, p.sketch_seed, mode="blendenpik", f=p.f, alpha=p.alpha)
    b = fab.solve(A, p.b, p.m, p.k, p.s, p.sketch_seed, mode="blendenpik", f=p.f, alpha=p.alpha,
                  precond=(4 * p.m, 12345))
    assert b["lsqr"]["iters"] < a["lsqr"]["iters"]
    assert rel(b["f_m"], a["f_m"]) <= 1e-8

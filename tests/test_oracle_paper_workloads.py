"""Oracle pins for the paper's dataset-free workloads:
sign(A) b by (A^2)^{-1/2} (A b), the 3D Laplacian inverse
square root (l.417-421) and the variable-coefficient convection-diffusion
exponential (l.366-374).  Each pin is something the oracle cannot reproduce
by re-running its own code: a closed form (eigen / sine-transform
decomposition), an independent library routine (scipy.linalg.signm,
scipy.sparse.linalg.expm_multiply) or an algebraic identity."""
import json
import os

import numpy as np
import pytest
import scipy.fft as sfft
import scipy.linalg as sl
import scipy.sparse as sp
import scipy.sparse.linalg as spl

import fab_problems as fp
from oracle import fab

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


# ---- sign(A) b = (A^2)^{-1/2} (A b) (l.406) ---------------------------------
def test_sign_golden_diag():
    # S:491 hand case: A = diag(2, -3), b = (1, 1) -> sign(A) b = (1, -1)
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["sign_diag"]
    A = sp.csr_matrix(np.array(g["A"], dtype=float))
    out = fab.sign(A, np.array(g["b"], dtype=float), 2, 2, 2, 1, mode="none")
    assert np.allclose(out["f_m"], g["signAb"], atol=1e-12)


@pytest.mark.parametrize("mode", fab.MODES)
def test_sign_symmetric_closed_form(mode):
    # A = Q diag(lam) Q^T with |lam| in [1, 3] of both signs: sign(A) b =
    # Q diag(sign lam) Q^T b exactly.  (A^2)^{-1/2} on [1, 9] converges like
    # 0.5^m, so m = 40 is converged to rounding.
    rng = np.random.default_rng(7)
    n = 128
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = rng.uniform(1.0, 3.0, n) * np.where(rng.random(n) < 0.5, -1.0, 1.0)
    A = (Q * lam) @ Q.T
    b = rng.standard_normal(n)
    exact = Q @ (np.sign(lam) * (Q.T @ b))
    out = fab.sign(A, b, 40, 2, 80, 11, mode=mode, lsqr_iters=60)
    assert rel(out["f_m"], exact) <= 1e-10, rel(out["f_m"], exact)


@pytest.mark.parametrize("whiten", [False, True])
def test_sign_nonsymmetric_matches_signm(whiten):
    # e4 recipe (nonnormal, spectrum in both half planes) against
    # scipy.linalg.signm (a different algorithm: Schur-based iteration)
    p = fp.make("e4", n=400, m=30, s=64)
    A = p.scipy()
    ref = sl.signm(A.toarray()) @ p.b
    out = fab.sign(A, p.b, p.m, p.k, p.s, p.sketch_seed, mode="blendenpik", whiten=whiten, lsqr_iters=60)
    assert rel(out["f_m"], ref) <= 1e-9, rel(out["f_m"], ref)


def test_sign_is_an_involution():
    # sign(A)^2 = I: applying the method to its own output returns b
    p = fp.make("e4", n=600, m=30, s=64)
    A = p.scipy()
    y = fab.sign(A, p.b, p.m, p.k, p.s, p.sketch_seed, mode="sketch_solve")["f_m"]
    z = fab.sign(A, y, p.m, p.k, p.s, p.sketch_seed, mode="sketch_solve")["f_m"]
    assert rel(z, p.b) <= 1e-9


def test_e4_spectrum_in_both_half_planes():
    A = fp.make("e4", n=500).scipy().toarray()
    ev = np.linalg.eigvals(A)
    assert (ev.real > 3).sum() > 100 and (ev.real < -3).sum() > 100
    assert np.abs(ev.real).min() > 3.0


# ---- 3D Laplacian, f = invsqrt (l.417-421) ----------------------------------
def dst_invsqrt(N, b):
    """Exact A^{-1/2} b for A = T (x) I (x) I + I (x) T (x) I + I (x) I (x) T,
    T = tridiag(-1, 2, -1) of size N: A = S diag(lam) S with S the orthonormal
    DST-I, lam_{ijk} = mu_i + mu_j + mu_k, mu_i = 2 - 2 cos(pi i / (N+1))."""
    mu = 2.0 - 2.0 * np.cos(np.pi * np.arange(1, N + 1) / (N + 1))
    lam = mu[:, None, None] + mu[None, :, None] + mu[None, None, :]
    B = b.reshape(N, N, N)
    C = sfft.dstn(B, type=1, norm="ortho")
    return sfft.idstn(C / np.sqrt(lam), type=1, norm="ortho").ravel()


def test_e5_generator_is_the_kronecker_laplacian():
    N = 5
    T = sp.diags([-np.ones(N - 1), 2 * np.ones(N), -np.ones(N - 1)], [-1, 0, 1])
    I = sp.identity(N)
    K = sp.kron(sp.kron(T, I), I) + sp.kron(sp.kron(I, T), I) + sp.kron(sp.kron(I, I), T)
    A = fp.make("e5", g=N, m=10).scipy()
    assert abs(A - K).max() == 0.0
    p = fp.make("e5", g=N, m=40)
    assert p.s == 42                                    # floor(1.05 m), l.421


def test_e5_dense_and_methods_match_dst_closed_form():
    N = 10
    p = fp.make("e5", g=N, m=80)
    A = p.scipy()
    exact = dst_invsqrt(N, p.b)
    assert rel(fab.dense(A, p.b, "invsqrt"), exact) <= 1e-12
    # kappa ~ 49: the Krylov approximants converge like ~0.75^m
    assert rel(fab.fom(A, p.b, 80, f="invsqrt"), exact) <= 1e-9
    out = fab.solve(A, p.b, 80, 2, p.s, p.sketch_seed, mode="none", f="invsqrt")
    assert rel(out["f_m"], exact) <= 1e-9
    a3 = fab.alg3(A, p.b, 80, p.s, p.sketch_seed, f="invsqrt", lsqr_iters=200)
    assert rel(a3["f_m"], exact) <= 1e-9


# ---- variable-coefficient convection-diffusion (l.366-374) ------------------
def test_e1_operator_structure():
    p = fp.make("e1", g=24, m=10)
    A = p.scipy()
    # the convection form 1/2 (v.grad u) + 1/2 div(v u) is skew-adjoint: the
    # symmetric part of A is the diffusion operator alone (row sums of its
    # off-diagonals = -centre on interior rows, SPD)
    S = ((A + A.T) / 2).toarray()
    assert np.linalg.eigvalsh(S).min() > 0
    g, h = 24, 1.0 / 25
    # D1 = 1000 inside [1/4, 3/4]^2, 1 outside; D2 = D1 / 2 (centre coefficient)
    centre = A.diagonal()
    assert np.isclose(centre[0], (1 + 1 + 0.5 + 0.5) / h ** 2)
    mid = (g // 2) * g + g // 2
    assert np.isclose(centre[mid], (1000 + 1000 + 500 + 500) / h ** 2)
    # b = sin(pi x) sin(pi y), normalized
    assert np.isclose(np.linalg.norm(p.b), 1.0)
    assert p.alpha == -1e3 / p.norm_inf                  # G-30


def test_e1_methods_match_expm_multiply():
    # all proposed methods "produce approximately the same result" (l.373):
    # against scipy's expm_multiply (truncated Taylor, an independent method).
    # Measured at g = 30 (rel. error vs expm_multiply): m = 70: FOM 1.5e-5,
    # Alg 5 1.8e-4, sketch-and-solve 2.4e-5, Blendenpik 1.5e-5; m = 90: 2.1e-7,
    # 1.8e-5, 3.6e-7, 2.1e-7.  Pinned: every method converges toward the
    # reference, Blendenpik with a (near-)exact LS solve equals FOM (Lemma 1).
    p = fp.make("e1", g=30, m=90, s=180)
    A = p.scipy()
    ref = spl.expm_multiply(p.alpha * A, p.b)
    fom = fab.fom(A, p.b, p.m, f="exp", alpha=p.alpha)
    assert rel(fom, ref) <= 1e-6
    errs = {}
    for mode in fab.MODES:
        out = fab.solve(A, p.b, p.m, p.k, p.s, p.sketch_seed, mode=mode, f="exp", alpha=p.alpha,
                        lsqr_iters=80)
        errs[mode] = rel(out["f_m"], ref)
        if mode == "blendenpik":
            assert rel(out["f_m"], fom) <= 1e-8
    assert errs["blendenpik"] <= 1e-6 and errs["sketch_solve"] <= 1e-5 and errs["none"] <= 1e-4, errs
    a3 = fab.alg3(A, p.b, p.m, p.s, p.sketch_seed, f="exp", alpha=p.alpha, lsqr_iters=200)
    assert rel(a3["f_m"], ref) <= 1e-6

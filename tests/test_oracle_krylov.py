"""Pins for oracle/krylov.py: Algorithm 2 and Arnoldi
(Eq. (2), l.38-48)."""
import json
import os

import numpy as np
import scipy.sparse as sp

import fab_problems as fp
from oracle import krylov

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _arnoldi_like_residual(A, V, H):
    m = H.shape[1]
    R = A @ V[:, :m] - V[:, : m + 1] @ H
    return np.linalg.norm(R) / (abs(A).sum(axis=1).max() * np.linalg.norm(V[:, :m]))


def test_stencil_matvec_hand_case():
    # tridiag(-1, 2, -1) (1, 1, 1) = (1, 0, 1)
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["tridiag_matvec"]
    ip, ix, dv = fp.stencil_csr((3, 1, 1), (2.0, -1.0, -1.0, 0, 0, 0, 0))
    A = sp.csr_matrix((dv, ix, ip), shape=(3, 3))
    assert np.array_equal(A @ np.array(g["x"]), np.array(g["y"]))


def test_symmetric_k2_is_lanczos():
    # l.104: for symmetric A and k = 2, Alg 2 coincides with Lanczos: H tridiagonal
    # and V orthonormal (in exact arithmetic; well-conditioned instance here)
    n = 400
    A = sp.diags([-np.ones(n - 1), 2 + np.linspace(0, 1, n), -np.ones(n - 1)], [-1, 0, 1]).tocsr()
    b = np.random.default_rng(0).standard_normal(n)
    d = krylov.truncated_arnoldi(A, b, 20, 2, variant="mgs")
    H, V = d["H"], d["V"]
    assert np.abs(np.triu(H[:20, :20], 2)).max() <= 1e-10 * np.abs(H).max()
    assert np.linalg.norm(V.T @ V - np.eye(21)) <= 1e-8
    assert np.allclose(H[:20, :20], H[:20, :20].T, atol=1e-10 * np.abs(H).max())


def test_k_ge_m_equals_full_arnoldi():
    # k >= m -> truncation inactive -> identical to Arnoldi (single pass MGS)
    # (well-conditioned Krylov basis, so single-pass MGS keeps orthogonality)
    p = fp.make("c1", g=20, m=15, k=2, s=40)
    A, b = p.scipy(), p.b
    d1 = krylov.truncated_arnoldi(A, b, 15, 15, variant="mgs")
    d2 = krylov.arnoldi(A, b, 15)
    assert np.allclose(d1["H"], d2["H"], rtol=0, atol=1e-10 * np.abs(d2["H"]).max())
    assert np.allclose(d1["V"], d2["V"], atol=1e-10)
    assert np.linalg.norm(d2["V"].T @ d2["V"] - np.eye(16)) <= 1e-12


def test_window_orthogonality_residual_unit_columns():
    p = fp.make("c3", g=20, m=40, k=4, s=80)
    A, b = p.scipy(), p.b
    d = krylov.truncated_arnoldi(A, b, 40, 4)
    V, H = d["V"], d["H"]
    G = V.T @ V
    for i in range(41):
        for j in range(max(0, i - 4), i):
            assert abs(G[i, j]) <= 1e-12                    # orthogonal to last k
    assert np.allclose(np.diag(G), 1.0, atol=1e-14)         # unit columns (l.126)
    assert _arnoldi_like_residual(A, V, H) <= 1e-12          # Eq. (3)
    assert np.linalg.norm(V[:, :40], 2) <= np.sqrt(40) + 1e-12   # l.337
    assert np.abs(np.tril(H, -2)).max() == 0.0               # upper Hessenberg
    # banded: column c has rows c+1-k..c+1 only (k-truncation)
    assert np.abs(np.triu(H, 4)).max() == 0.0


def test_mgs_equals_cgs_within_window():
    # G-2: CGS and MGS agree (window is orthonormal)
    p = fp.make("c1", g=30, m=25, k=2, s=50)
    A, b = p.scipy(), p.b
    a = krylov.truncated_arnoldi(A, b, 25, 2, variant="mgs")
    c = krylov.truncated_arnoldi(A, b, 25, 2, variant="cgs")
    assert np.abs(a["H"] - c["H"]).max() <= 1e-11 * np.abs(a["H"]).max()
    assert np.abs(a["V"] - c["V"]).max() <= 1e-10


def test_breakdown_eigenvector():
    # A = diag(1..5), b = e_1 -> breakdown at i = 2, H = [1]
    A = sp.diags(np.arange(1.0, 6.0)).tocsr()
    b = np.zeros(5)
    b[0] = 1
    d = krylov.truncated_arnoldi(A, b, 3, 2)
    assert d["breakdown"] and d["m_eff"] == 1
    assert d["H"][0, 0] == 1.0
    d = krylov.arnoldi(A, b, 3)
    assert d["breakdown"] and d["m_eff"] == 1


def test_breakdown_distinct_eigenvalues():
    # diagonal A with d distinct values: Krylov space of dimension d
    A = sp.diags(np.repeat([1.0, 2.0, 3.0, 4.0], 10)).tocsr()
    b = np.random.default_rng(1).standard_normal(40)
    d = krylov.truncated_arnoldi(A, b, 10, 10)
    assert d["breakdown"] and d["m_eff"] == 4


# ---- Algorithm 1 (sketched Gram-Schmidt) ---------------
def _srht(n, s, seed=1):
    from oracle.srht import SRHT
    return SRHT(n, s, seed)


def test_sketched_gs_sketch_orthonormal_and_arnoldi_like():
    # l.94: S_i stays orthonormal by construction; l.97 / Eq. (3): A V_m = V_{m+1} H_m
    # (a problem whose Krylov space is not yet saturated at m: with r_ii << ||p_i||
    # one CGS pass loses sketch orthogonality, as for any single-pass GS)
    p = fp.make("c1", g=40, m=30, k=2, s=70)
    A = p.scipy()
    d = krylov.sketched_gs(A, p.b, p.m, _srht(p.n, p.s, 7))
    S, V, H = d["S"], d["V"], d["H"]
    # one CGS pass per step: orthogonality holds to ~eps ||p_i|| / r_ii (here
    # r_ii / ||p_i|| ~ 1e-3 late in the run), so 1e-10, not machine precision
    assert np.abs(S.T @ S - np.eye(p.m + 1)).max() <= 1e-10
    assert _arnoldi_like_residual(A, V, H) <= 1e-13
    assert np.allclose(H, np.triu(H, -1))                     # upper Hessenberg
    th = _srht(p.n, p.s, 7)
    assert np.abs(th.apply(V) - S).max() <= 1e-12             # S = Theta V (the sketch is exact)
    assert abs(d["gamma"] - np.linalg.norm(th.apply(p.b))) <= 1e-14 * d["gamma"]
    assert np.linalg.cond(V) <= 10.0                          # well-conditioned (Balabanov-Grigori Prop 4.1)


def test_sketched_gs_with_orthogonal_sketch_is_arnoldi():
    # s = N = n: Theta = (1/sqrt N) H_N D is orthogonal, so sketched GS is exact
    # Gram-Schmidt: V orthonormal and underline-H = Arnoldi's (up to rounding)
    n = 256
    A = sp.diags([np.full(n - 1, -1.0), 2 + np.linspace(0, 3, n), np.full(n - 1, -0.5)], [-1, 0, 1]).tocsr()
    b = np.random.default_rng(3).standard_normal(n)
    d = krylov.sketched_gs(A, b, 12, _srht(n, n, 11))
    ref = krylov.arnoldi(A, b, 12)
    assert np.abs(d["V"].T @ d["V"] - np.eye(13)).max() <= 1e-12
    assert np.abs(d["H"] - ref["H"]).max() <= 1e-12 * np.abs(ref["H"]).max()
    assert np.abs(d["V"] - ref["V"]).max() <= 1e-12
    assert abs(d["gamma"] - np.linalg.norm(b)) <= 1e-13 * np.linalg.norm(b)


def test_sketched_gs_breakdown_distinct_eigenvalues():
    vals = np.repeat([1.0, 2.0, 3.5, 5.0], 64)
    A = sp.diags(vals).tocsr()
    b = np.random.default_rng(4).standard_normal(len(vals))
    d = krylov.sketched_gs(A, b, 10, _srht(len(vals), 24, 2))
    assert d["breakdown"] and d["m_eff"] == 4


# ---- Algorithm 2 with whitening ----------------
def test_whitening_restores_a_well_conditioned_basis():
    # c4 (power-law graph): the truncated basis goes numerically rank-deficient
    # (cond ~1e15 by m = 50); whitening at cond > 1000 keeps it
    # well-conditioned and the Arnoldi-like relation / V^+ b = gamma e_1 hold
    p = fp.make("c4", n=1 << 13, m=60, k=2, s=130)
    A = p.scipy()
    th = _srht(p.n, p.s, p.sketch_seed)
    plain = krylov.truncated_arnoldi(A, p.b, p.m, p.k, variant="mgs")
    assert np.linalg.cond(plain["V"]) > 1e8
    d = krylov.whitened_basis(A, p.b, p.m, p.k, th)
    V, H = d["V"], d["H"]
    assert 2 < d["whitened_at"] <= p.m
    assert np.linalg.cond(V) <= 20
    assert _arnoldi_like_residual(A, V, H) <= 1e-13
    S = th.apply(V)
    assert np.abs(S.T @ S - np.eye(p.m + 1)).max() <= 1e-10      # orthonormal sketch after whitening
    coef = np.linalg.lstsq(V[:, : p.m], p.b, rcond=None)[0]
    assert np.abs(coef - d["gamma"] * np.eye(p.m)[0]).max() <= 1e-12 * d["gamma"]


def test_whitening_never_triggered_is_algorithm2():
    p = fp.make("c3", g=16, m=30, k=4, s=70)
    A = p.scipy()
    d = krylov.whitened_basis(A, p.b, p.m, p.k, _srht(p.n, p.s, 1), cond_max=np.inf)
    ref = krylov.truncated_arnoldi(A, p.b, p.m, p.k, variant="mgs")
    assert d["whitened_at"] == 0
    assert np.array_equal(d["V"], ref["V"]) and np.array_equal(d["H"], ref["H"])


def test_whitening_at_first_check_is_algorithm1_remark():
    # Remark after Alg 2 (l.109): Alg 1 = Alg 2 followed by whitening.  Whitening
    # at the first check (V_2) and continuing with Alg 1 reproduces Alg 1 (the
    # QR factor with positive diagonal is unique)
    p = fp.make("c1", g=30, m=20, k=2, s=50)
    A = p.scipy()
    th = _srht(p.n, p.s, 4)
    d = krylov.whitened_basis(A, p.b, p.m, p.k, th, cond_max=0.0)
    ref = krylov.sketched_gs(A, p.b, p.m, th)
    assert d["whitened_at"] == 2
    assert np.abs(d["V"] - ref["V"]).max() <= 1e-10 * np.abs(ref["V"]).max()
    assert np.abs(d["H"] - ref["H"]).max() <= 1e-10 * np.abs(ref["H"]).max()
    assert abs(d["gamma"] - ref["gamma"]) <= 1e-12 * ref["gamma"]


def test_cond1_upper_closed_form():
    R = np.array([[2.0, 1.0], [0.0, 0.5]])
    # ||R||_1 = 2.0 (col 0: 2, col 1: 1.5); R^-1 = [[0.5, -1], [0, 2]] -> ||.||_1 = 3
    assert krylov.cond1_upper(R) == 6.0

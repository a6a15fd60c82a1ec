"""Pins for oracle/lsq.py and oracle/matfun.py (§3.1.1, l.174-184,
Remark 2 l.249-251, l.356)."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import lsq, matfun, srht

GOLD = os.path.join(os.path.dirname(__file__), "golden")
G = json.load(open(os.path.join(GOLD, "spec_examples.json")))


def test_qr_hand_case():
    g = G["qr_3_4"]
    R, Qt = lsq.householder_qr(np.array(g["A"]), np.eye(2))
    assert np.allclose(R, g["R"], atol=1e-15)
    Q = Qt.T[:, :1]
    assert np.allclose(Q, g["Q"], atol=1e-15)


def test_qr_matches_numpy_with_sign_convention():
    rs = np.random.default_rng(0)
    for shape in [(20, 5), (600, 300), (7, 7)]:
        A = rs.standard_normal(shape)
        A[:, 0] *= -1
        R, Qt = lsq.householder_qr(A, np.eye(shape[0]))
        assert np.all(np.diag(R) >= 0)
        Qn, Rn = np.linalg.qr(A)
        sg = np.sign(np.diag(Rn))
        assert np.allclose(R, sg[:, None] * Rn, atol=1e-12 * np.abs(A).max())
        Q = Qt.T[:, : shape[1]]
        assert np.allclose(Q @ R, A, atol=1e-12 * np.abs(A).max())
        assert np.allclose(Qt @ Qt.T, np.eye(shape[0]), atol=1e-12)


def test_qr_zero_and_negative_columns():
    A = np.array([[-2.0, 1.0], [0.0, 3.0], [0.0, 4.0]])
    R, _ = lsq.householder_qr(A)
    assert np.allclose(R, [[2.0, -1.0], [0.0, 5.0]])


def test_trsv_hand_case_and_singular():
    g = G["trsv"]
    assert np.allclose(lsq.solve_upper(np.array(g["R"]), np.array(g["b"])), g["x"])
    R = np.array([[1.0, 2.0], [0.0, 0.0]])
    with pytest.raises(lsq.SingularTriangular):
        lsq.solve_upper(R, np.ones(2))
    R = np.triu(np.random.default_rng(1).standard_normal((6, 6))) + 6 * np.eye(6)
    b = np.arange(6.0)
    assert np.allclose(R.T @ lsq.solve_upper_transposed(R, b), b)


def test_lsqr_matches_lstsq():
    rs = np.random.default_rng(2)
    V = rs.standard_normal((500, 20)) @ np.diag(np.linspace(1, 5, 20))
    c = rs.standard_normal(500)
    ystar = np.linalg.lstsq(V, c, rcond=None)[0]
    y, info = lsq.lsqr(lambda v: V @ v, lambda u: V.T @ u, c, 20, tol=1e-14, maxit=200)
    assert np.linalg.norm(y - ystar) <= 1e-10 * np.linalg.norm(ystar)
    # orthonormal V: solution = V^T c
    Q, _ = np.linalg.qr(V)
    y, _ = lsq.lsqr(lambda v: Q @ v, lambda u: Q.T @ u, c, 20, tol=1e-14)
    assert np.allclose(y, Q.T @ c, atol=1e-12)
    # square identity: y = c
    y, info = lsq.lsqr(lambda v: v, lambda u: u, c[:20], 20, tol=1e-12)
    assert np.allclose(y, c[:20]) and info["iters"] <= 2


def test_lsqr_residual_monotone():
    rs = np.random.default_rng(3)
    V = rs.standard_normal((300, 15))
    c = rs.standard_normal(300)
    prev = np.inf
    for L in range(1, 15):
        y, _ = lsq.lsqr(lambda v: V @ v, lambda u: V.T @ u, c, 15, iters=L)
        r = np.linalg.norm(V @ y - c)
        assert r <= prev + 1e-12
        prev = r


def test_blendenpik_ill_conditioned():
    # cond(V) = 1e6: preconditioned LSQR converges in <= 60 iterations,
    # plain LSQR is >= 10x worse at the same count
    rs = np.random.default_rng(4)
    n, m = 2048, 20
    Q, _ = np.linalg.qr(rs.standard_normal((n, m)))
    W, _ = np.linalg.qr(rs.standard_normal((m, m)))
    V = Q @ np.diag(np.logspace(0, -6, m)) @ W
    c = rs.standard_normal(n)
    ystar = np.linalg.lstsq(V, c, rcond=None)[0]
    th = srht.SRHT(n, 2 * m, seed=5)
    y, R, info = lsq.blendenpik(V, c, th.apply(V), iters=60)
    yp, _ = lsq.lsqr(lambda v: V @ v, lambda u: V.T @ u, c, m, iters=60)
    e_b = np.linalg.norm(y - ystar) / np.linalg.norm(ystar)
    e_p = np.linalg.norm(yp - ystar) / np.linalg.norm(ystar)
    assert e_b <= 1e-8 and e_p >= 10 * e_b


def test_sketch_and_solve_orthogonal_sketch_is_exact():
    # s = N (orthogonal Theta) -> exact least squares; c _|_ range -> 0
    rs = np.random.default_rng(6)
    n, m = 256, 10
    V = rs.standard_normal((n, m))
    c = rs.standard_normal(n)
    th = srht.SRHT(n, n, seed=7)
    y, _ = lsq.sketch_and_solve(th.apply(V), th.apply(c))
    assert np.allclose(y, np.linalg.lstsq(V, c, rcond=None)[0], atol=1e-12)
    Q, _ = np.linalg.qr(V, mode="complete")
    cp = Q[:, m:] @ rs.standard_normal(n - m)
    y, _ = lsq.sketch_and_solve(th.apply(V), th.apply(cp))
    assert np.abs(y).max() <= 1e-12


@pytest.mark.parametrize("key,f", [("expm_nilpotent", "exp"), ("expm_diag", "exp"),
                                   ("sqrtm_jordan", "sqrt"), ("sqrtm_diag", "sqrt"),
                                   ("invsqrtm_diag", "invsqrt")])
def test_matfun_hand_cases(key, f):
    g = G[key]
    A = np.array(g["A"])
    F = np.array(g["F"])
    assert np.allclose(matfun.fmat(f, A), F, rtol=1e-14, atol=1e-14)
    assert np.allclose(matfun.f_e1(f, A), F[:, 0], rtol=1e-14, atol=1e-14)


def test_matfun_identities():
    rs = np.random.default_rng(8)
    for _ in range(5):
        H = rs.standard_normal((30, 30))
        H *= 5 / np.linalg.norm(H, 2)
        E = matfun.fmat("exp", H)
        assert np.allclose(E @ matfun.fmat("exp", -H), np.eye(30), atol=1e-10)
        assert np.linalg.norm(E @ H - H @ E) <= 1e-9 * np.linalg.norm(H) * np.linalg.norm(E)
        P = H @ H.T + 30 * np.eye(30) + 0.5 * H          # eigenvalues in right half plane
        X = matfun.fmat("sqrt", P)
        assert np.linalg.norm(X @ X - P) <= 1e-12 * np.linalg.norm(P)
        Y = matfun.fmat("invsqrt", P)
        assert np.linalg.norm(Y @ X - np.eye(30)) <= 1e-11
    # poly kind: Horner vs explicit powers
    A = rs.standard_normal((6, 6))
    assert np.allclose(matfun.fmat("poly", A, poly=[1, 2, 3]), np.eye(6) + 2 * A + 3 * A @ A)
    with pytest.raises(matfun.DomainError):
        matfun.fmat("sqrt", np.diag([1.0, -2.0]))


def test_expm_against_taylor():
    # S:226 style: scaled Taylor series oracle
    rs = np.random.default_rng(9)
    H = rs.standard_normal((20, 20))
    H *= 3 / np.linalg.norm(H, 1)
    X = H / 16
    T = np.eye(20)
    term = np.eye(20)
    for j in range(1, 40):
        term = term @ X / j
        T = T + term
    for _ in range(4):
        T = T @ T
    assert np.allclose(matfun.fmat("exp", H), T, rtol=1e-12, atol=1e-12)
    assert np.allclose(matfun.fmat("exp", H), sla.expm(H), rtol=1e-13, atol=1e-14)

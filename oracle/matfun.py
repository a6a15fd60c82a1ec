"""Small dense matrix functions f(X) e_1 on the compressed matrix
("For the evaluation of f on the compressed matrices we used
Matlab expm and sqrtm functions").  The oracle uses the corresponding library
primitives: scipy.linalg.expm (scaling and squaring with Pade, Al-Mohy &
Higham, as MATLAB's expm) and scipy.linalg.sqrtm (Schur method, as MATLAB's
sqrtm).  The inverse square root is sqrtm(X)^{-1} e_1 by an LU solve (SPEC
S:237-240).  f is applied to X = alpha*C + sigma*I (reading G-17: the configs
ask for exp(-tA), sqrt(A + sigma I), (-A)^{-1/2}; V^+(alpha A + sigma I)V =
alpha C + sigma I because the Krylov space is shift-invariant).  'poly' is
the test-only polynomial kind for the exactness pin.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np
import scipy.linalg as sla


class DomainError(ValueError):
    pass


def _check_sqrt_domain(X):
    ev = np.linalg.eigvals(X)
    bad = (np.abs(ev.imag) <= 1e-12 * max(1.0, np.abs(ev).max())) & (ev.real <= 0)
    if bad.any():
        raise DomainError("eigenvalue on the closed negative real axis")


def fmat(f: str, X: np.ndarray, poly=None) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if f == "exp":
        return sla.expm(X)
    if f in ("sqrt", "invsqrt"):
        _check_sqrt_domain(X)
        S = sla.sqrtm(X)
        if np.iscomplexobj(S):
            S = S.real
        if f == "sqrt":
            return S
        return np.linalg.solve(S, np.eye(X.shape[0]))
    if f == "poly":
        # Horner: p(X) = sum_i poly[i] X^i
        P = np.zeros_like(X)
        I = np.eye(X.shape[0])
        for a in reversed(list(poly)):
            P = P @ X + a * I
        return P
    raise ValueError(f)


def f_e1(f: str, C: np.ndarray, alpha: float = 1.0, sigma: float = 0.0,
         poly=None) -> np.ndarray:
    """c = f(alpha C + sigma I) e_1."""
    m = C.shape[0]
    X = alpha * np.asarray(C, dtype=np.float64) + sigma * np.eye(m)
    if f == "invsqrt":
        _check_sqrt_domain(X)
        S = sla.sqrtm(X)
        if np.iscomplexobj(S):
            S = S.real
        e1 = np.zeros(m)
        e1[0] = 1.0
        return np.linalg.solve(S, e1)
    return fmat(f, X, poly)[:, 0]


def f_dense_apply(f: str, A: np.ndarray, b: np.ndarray, alpha=1.0, sigma=0.0,
                  poly=None) -> np.ndarray:
    """Dense reference f(alpha A + sigma I) b for small n (PAPER.md l.358:
    'exact' value via expm/sqrtm when n < 1e4)."""
    n = A.shape[0]
    X = alpha * np.asarray(A, dtype=np.float64) + sigma * np.eye(n)
    if f == "invsqrt":
        _check_sqrt_domain(X)
        S = sla.sqrtm(X)
        S = S.real if np.iscomplexobj(S) else S
        return np.linalg.solve(S, b)
    return fmat(f, X, poly) @ b

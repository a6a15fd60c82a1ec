"""Least-squares pieces for the compression (§3.1.1, l.174-184,
and Remark 2, l.249-251):

  Eq. (7)   y = argmin_z || V_m z - v_{m+1} ||_2
  Blendenpik (l.183): "computes a random sketch of the basis using, once
            again, a SRHT, and then uses the R factor from a QR decomposition
            of the sketch as a preconditioner" -> LSQR on V_m R^{-1}.
  Remark 2: sketch-and-solve  y = argmin_z || Theta (V_m z - v_{m+1}) ||_2.

Householder QR with R_ii >= 0 (Golub & Van Loan Alg. 5.1.1 'house' with
P x = ||x|| e_1), back substitution, and LSQR (Paige & Saunders 1982) with
x_0 = 0 and the MATLAB `lsqr` stopping test the paper used (l.359, tol 1e-6):
stop when ||r||/||b|| <= tol or ||M^T r|| / (||M||_F ||r||) <= tol (reading
G-14); `iters=L` instead runs exactly L iterations (parity mode).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import math

import numpy as np


class SingularTriangular(ValueError):
    pass


def house(x: np.ndarray):
    """v (v[0] = 1), beta, mu with (I - beta v v^T) x = mu e_1, mu = ||x||."""
    x = np.asarray(x, dtype=np.float64)
    sigma = float(x[1:] @ x[1:])
    v = x.copy()
    v[0] = 1.0
    x0 = float(x[0])
    if sigma == 0.0:
        return v, (0.0 if x0 >= 0 else 2.0), abs(x0)
    mu = math.sqrt(x0 * x0 + sigma)
    v0 = x0 - mu if x0 <= 0 else -sigma / (x0 + mu)
    beta = 2.0 * v0 * v0 / (sigma + v0 * v0)
    v = x / v0
    v[0] = 1.0
    return v, beta, mu


def householder_qr(A: np.ndarray, C: np.ndarray = None):
    """R (ncol x ncol, R_ii >= 0) of A = QR and Q^T C (all rows) if C given."""
    A = np.array(A, dtype=np.float64, copy=True)
    rows, cols = A.shape
    if rows < cols:
        raise ValueError("need rows >= cols")
    QtC = None if C is None else np.array(C, dtype=np.float64).reshape(rows, -1).copy()
    for j in range(cols):
        v, beta, mu = house(A[j:, j])
        if beta != 0.0:
            A[j:, j + 1:] -= beta * np.outer(v, v @ A[j:, j + 1:])
            if QtC is not None:
                QtC[j:] -= beta * np.outer(v, v @ QtC[j:])
        A[j, j] = mu
        A[j + 1:, j] = 0.0
    if QtC is not None:
        QtC = QtC.reshape(np.shape(C))
    return np.triu(A[:cols, :]), QtC


def solve_upper(R: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Back substitution R X = B (SingularTriangular when
    |r_jj| < 1e-14 max |r_ii|)."""
    R = np.asarray(R, dtype=np.float64)
    d = np.abs(np.diag(R))
    if d.size and d.min() < 1e-14 * d.max():
        raise SingularTriangular("singular triangular factor")
    X = np.array(B, dtype=np.float64, copy=True)
    m = R.shape[0]
    for i in range(m - 1, -1, -1):
        X[i] = (X[i] - R[i, i + 1:] @ X[i + 1:]) / R[i, i]
    return X


def solve_upper_transposed(R: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Forward substitution R^T X = B."""
    R = np.asarray(R, dtype=np.float64)
    X = np.array(B, dtype=np.float64, copy=True)
    m = R.shape[0]
    for i in range(m):
        X[i] = (X[i] - R[:i, i] @ X[:i]) / R[i, i]
    return X


def lsqr(matvec, rmatvec, b: np.ndarray, ncols: int, tol: float = 1e-6,
         maxit: int = None, iters: int = None):
    """LSQR (Golub-Kahan bidiagonalization), x_0 = 0.
    Returns (x, info) with info = dict(iters, rnorm, arnorm, anorm)."""
    if maxit is None:
        maxit = 4 * ncols
    nit = iters if iters is not None else maxit
    x = np.zeros(ncols)
    beta = float(np.linalg.norm(b))
    info = dict(iters=0, rnorm=beta, arnorm=0.0, anorm=0.0, converged=False)
    if beta == 0.0:
        return x, info
    bnorm = beta
    u = b / beta
    v = rmatvec(u)
    alpha = float(np.linalg.norm(v))
    if alpha == 0.0:
        return x, info
    v = v / alpha
    w = v.copy()
    phibar, rhobar = beta, alpha
    anorm2 = 0.0
    it = 0
    for it in range(1, nit + 1):
        u = matvec(v) - alpha * u
        beta = float(np.linalg.norm(u))
        if beta > 0.0:
            u = u / beta
        anorm2 += alpha * alpha + beta * beta
        v = rmatvec(u) - beta * v
        alpha = float(np.linalg.norm(v))
        if alpha > 0.0:
            v = v / alpha
        rho = math.hypot(rhobar, beta)
        c, s = rhobar / rho, beta / rho
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        x = x + (phi / rho) * w
        w = v - (theta / rho) * w
        rnorm = phibar
        arnorm = phibar * alpha * abs(c)
        anorm = math.sqrt(anorm2)
        info.update(iters=it, rnorm=rnorm, arnorm=arnorm, anorm=anorm)
        if alpha == 0.0 or beta == 0.0:
            # the bidiagonalization terminated: x is the exact LS solution (the
            # algorithm stops here in every mode, MATLAB lsqr as well)
            info["converged"] = True
            break
        if iters is None:
            if rnorm / bnorm <= tol or (rnorm > 0 and arnorm / (anorm * rnorm) <= tol) \
                    or alpha == 0.0 or beta == 0.0:
                info["converged"] = True
                break
    return x, info


def blendenpik(Vm: np.ndarray, c: np.ndarray, SVm: np.ndarray, tol=1e-6,
               maxit=None, iters=None, rinv="solve"):
    """argmin ||Vm z - c|| by LSQR right-preconditioned with R from the QR
    of the sketch SVm = Theta Vm.  Returns (y, R, info).
    rinv="inverse" applies R^{-1} as an explicit inverse instead of by
    substitution: the same method in different rounding, used only to
    measure the rounding sensitivity of intermediate LSQR iterates."""
    R, _ = householder_qr(SVm)
    m = R.shape[0]
    if rinv == "inverse":
        Ri = solve_upper(R, np.eye(m))
        mv = lambda p: Vm @ (Ri @ p)
        rmv = lambda u: Ri.T @ (Vm.T @ u)
    else:
        mv = lambda p: Vm @ solve_upper(R, p)                   # (Vm R^-1) p
        rmv = lambda u: solve_upper_transposed(R, Vm.T @ u)     # R^-T Vm^T u
    z, info = lsqr(mv, rmv, c, m, tol=tol, maxit=maxit, iters=iters)
    return solve_upper(R, z), R, info


def sketch_and_solve(SVm: np.ndarray, Sc: np.ndarray):
    """Remark 2: argmin_z ||Theta Vm z - Theta c|| via Householder QR of
    Theta Vm (y = R^{-1} (Q^T Theta c)[:m]).  Returns (y, R)."""
    R, QtSc = householder_qr(SVm, Sc)
    m = R.shape[0]
    return solve_upper(R, QtSc[:m]), R

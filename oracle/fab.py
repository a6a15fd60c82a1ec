"""f(A)b drivers (§3).

  alg4   Algorithm 4 (l.199-209): Alg 2 basis, y by Blendenpik, return
         ||b|| V_m f(H_m + h_{m+1,m} y e_m^T) e_1
  alg3   Algorithm 3 (l.187-197): Alg 1 basis, y by (plain) LSQR, return
         r_11 V_m f(H_m + h_{m+1,m} y e_m^T) e_1
  ss     Remark 2 (l.249-251): as Alg 4 with y from sketch-and-solve
         (mathematically sFOM, Eq. (9))
  alg5   Algorithm 5 (l.219-228): ||b|| V_m f(H_m) e_1, no least squares
  sfom   the literal Eq. (9) formula (cross-check of `ss`)
  fom    Eq. (4) with a full Arnoldi basis (the paper's baseline 'Arnoldi')
  dense  f(A) b formed densely (small n only)
  sign   sign(A) b by the formula of l.406, (A^2)^{-1/2} (A b): any of the
         above on the operator A^2 with the start vector A b, f = invsqrt

Compression (Eq. (6), l.167-171): V_m^+ A V_m = H_m + h_{m+1,m} (V_m^+ v_{m+1})
e_m^T, gamma_b = ||b||_2 for Alg 2 (l.172).  f is applied as
f(alpha C + sigma I) (reading G-17).  Reading G-12: Blendenpik reuses the
basis sketch Theta (one fab_sketch call), so SV_{m+1} = Theta V_{m+1} feeds
both the Blendenpik R and sketch-and-solve -- unless `precond=(s2, seed2)`
asks for Blendenpik's own sketch Theta' of V_m.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

from . import krylov, lsq, matfun
from .srht import SRHT

MODES = ("blendenpik", "sketch_solve", "none")


def compress(dec, SV, mode, lsqr_tol=1e-6, lsqr_iters=None, lsqr_maxit=None, rinv="solve", precond=None):
    """y and C_m = H_m + h_{m+1,m} y e_m^T from an Alg 2 decomposition.
    precond=(s2, seed2): Blendenpik takes its preconditioner from its own
    SRHT Theta' = SRHT(n, s2, seed2) of V_m ("computes a
    random sketch of the basis using, once again, a SRHT"; reading G-12's
    precond_s / precond_seed) instead of reusing SV = Theta V."""
    V, H, m = dec["V"], dec["H"], dec["m_eff"]
    Hm = H[:m, :m].copy()
    info = {}
    if dec["breakdown"] or mode == "none":
        y = np.zeros(m)
        R = None
        if mode != "none" and SV is not None:
            R, _ = lsq.householder_qr(SV[:, :m])
    elif mode == "blendenpik":
        SVp = SV[:, :m]
        if precond is not None:
            SVp = SRHT(V.shape[0], precond[0], precond[1]).apply(V[:, :m])      # Theta' V_m
        y, R, info = lsq.blendenpik(V[:, :m], V[:, m], SVp, tol=lsqr_tol,
                                    maxit=lsqr_maxit, iters=lsqr_iters, rinv=rinv)
    elif mode == "sketch_solve":
        y, R = lsq.sketch_and_solve(SV[:, :m], SV[:, m])
    else:
        raise ValueError(mode)
    C = Hm.copy()
    if not dec["breakdown"]:
        C[:, m - 1] += H[m, m - 1] * y                      # Eq. (6)
    return y, C, R, info


def solve(A, b, m, k, s, seed, mode="blendenpik", f="exp", alpha=1.0,
          sigma=0.0, poly=None, lsqr_tol=1e-6, lsqr_iters=None,
          lsqr_maxit=None, variant="cgs", keep=True, lsqr_rinv="solve", precond=None):
    """One f(A)b approximation by Alg 4 / Remark 2 / Alg 5.  Returns a dict
    with f_m and every intermediate (V, H, SV, rows, signs, y, C, c)."""
    dec = krylov.truncated_arnoldi(A, b, m, k, variant=variant)     # Alg 2
    me = dec["m_eff"]
    th = SV = None
    if mode != "none":
        th = SRHT(b.shape[0], s, seed)                              # Theta
        if me + 1 > s:
            raise ValueError("InvalidSketchSize: need s >= m+1")
        SV = th.apply(dec["V"])                                     # Theta V_{m+1}
    y, C, R, info = compress(dec, SV, mode, lsqr_tol, lsqr_iters, lsqr_maxit, lsqr_rinv, precond)
    c = matfun.f_e1(f, C, alpha, sigma, poly)                       # f(C) e_1
    fm = dec["gamma"] * (dec["V"][:, :me] @ c)                      # ||b|| V_m c
    out = dict(f_m=fm, H=dec["H"], gamma=dec["gamma"], m_eff=me,
               breakdown=dec["breakdown"], y=y, C=C, c=c, R=R, lsqr=info)
    if keep:
        out.update(V=dec["V"], SV=SV)
    if th is not None:
        out.update(rows=th.rows, signs=th.signs)
    return out


def sfom(A, b, m, k, s, seed, f="exp", alpha=1.0, sigma=0.0, poly=None):
    """Eq. (9) written out: Theta V_m = S_m R_m (thin QR),
    f_hat = V_m (R_m^{-1} f(S_m^T Theta A V_m R_m^{-1}) S_m^T Theta b)."""
    dec = krylov.truncated_arnoldi(A, b, m, k)
    me = dec["m_eff"]
    Vm = dec["V"][:, :me]
    th = SRHT(b.shape[0], s, seed)
    TV = th.apply(Vm)
    TAV = th.apply(A @ Vm)
    Tb = th.apply(b)
    Q, R = np.linalg.qr(TV)
    sg = np.sign(np.diag(R))
    Q, R = Q * sg, sg[:, None] * R
    Rinv = lsq.solve_upper(R, np.eye(me))
    inner = Q.T @ TAV @ Rinv
    F = matfun.fmat(f, alpha * inner + sigma * np.eye(me), poly) if f != "invsqrt" \
        else np.linalg.inv(matfun.fmat("sqrt", alpha * inner + sigma * np.eye(me)))
    return Vm @ (Rinv @ (F @ (Q.T @ Tb)))


def fom(A, b, m, f="exp", alpha=1.0, sigma=0.0, poly=None):
    """Eq. (4): f_m = ||b|| U_m f(K_m) e_1 with a full Arnoldi basis."""
    dec = krylov.arnoldi(A, b, m)
    me = dec["m_eff"]
    c = matfun.f_e1(f, dec["H"][:me, :me], alpha, sigma, poly)
    return dec["gamma"] * (dec["V"][:, :me] @ c)


def dense(A, b, f="exp", alpha=1.0, sigma=0.0, poly=None):
    Ad = A.toarray() if hasattr(A, "toarray") else np.asarray(A)
    return matfun.f_dense_apply(f, Ad, b, alpha, sigma, poly)


def alg3(A, b, m, s, seed, f="exp", alpha=1.0, sigma=0.0, poly=None, lsqr_tol=1e-6,
         lsqr_iters=None, mode="lsqr"):
    """Algorithm 3: basis by Algorithm 1 with the SRHT
    Theta (l.70; the same Theta as fab_sketch(s, seed)), y = argmin ||V_m z
    - v_{m+1}|| by LSQR (l.182: "a few iterations of LSQR ... is sufficient"
    for the well-conditioned BG basis), f_m = r_11 V_m f(C_m) e_1 (l.195).
    mode "none" skips the least squares (y = 0).  Returns a dict like solve."""
    th = SRHT(b.shape[0], s, seed)
    dec = krylov.sketched_gs(A, b, m, th)
    me = dec["m_eff"]
    V, H = dec["V"], dec["H"]
    y = np.zeros(me)
    info = {}
    if not dec["breakdown"] and mode == "lsqr":
        Vm, c = V[:, :me], V[:, me]
        y, info = lsq.lsqr(lambda z: Vm @ z, lambda u: Vm.T @ u, c, me, tol=lsqr_tol,
                           iters=lsqr_iters)                               # l.194
    C = H[:me, :me].copy()
    if not dec["breakdown"]:
        C[:, me - 1] += H[me, me - 1] * y                                   # Eq. (6)
    cvec = matfun.f_e1(f, C, alpha, sigma, poly)
    fm = dec["gamma"] * (V[:, :me] @ cvec)                                  # l.195
    return dict(f_m=fm, V=V, H=H, S=dec["S"], R=dec["R"], gamma=dec["gamma"], m_eff=me,
                breakdown=dec["breakdown"], y=y, C=C, c=cvec, lsqr=info, rows=th.rows,
                signs=th.signs)


def solve_whitened(A, b, m, k, s, seed, mode="blendenpik", f="exp", alpha=1.0, sigma=0.0, poly=None,
                   cond_max=1000.0, lsqr_tol=1e-6, lsqr_iters=None):
    """Algorithm 4 / Remark 2 / Algorithm 5 on the whitened basis (Algorithm 2
    with whitening at cond > cond_max, then Algorithm 1; PAPER.md l.106,
    l.395, l.457-458), f_m = gamma V_m f(C_m) e_1."""
    th = SRHT(b.shape[0], s, seed)
    dec = krylov.whitened_basis(A, b, m, k, th, cond_max=cond_max)
    me = dec["m_eff"]
    SV = th.apply(dec["V"]) if mode != "none" else None
    y, C, R, info = compress(dec, SV, mode, lsqr_tol, lsqr_iters, None)
    c = matfun.f_e1(f, C, alpha, sigma, poly)
    fm = dec["gamma"] * (dec["V"][:, :me] @ c)
    return dict(f_m=fm, V=dec["V"], H=dec["H"], SV=SV, gamma=dec["gamma"], m_eff=me,
                breakdown=dec["breakdown"], whitened_at=dec["whitened_at"], y=y, C=C, c=c, lsqr=info)


def sign(A, b, m, k, s, seed, mode="blendenpik", whiten=False, cond_max=1000.0, lsqr_tol=1e-6,
         lsqr_iters=None, keep=True):
    """sign(A) b ("to apply the sign function to a vector we
    use the formula f(A)b = (A^2)^{-1/2} (Ab)", Higham 2008 Ch. 5): the
    method -- Algorithm 4 / Remark 2 / Algorithm 5 on the Algorithm 2 basis,
    or on the whitened basis (l.395-406: the paper's sign example needs
    whitening) -- applied to the operator A^2 (formed as a sparse product)
    and the vector A b, with f = invsqrt (alpha = 1, sigma = 0)."""
    A2 = A @ A
    if hasattr(A2, "tocsr"):
        A2 = A2.tocsr()
    Ab = A @ b
    if whiten:
        return solve_whitened(A2, Ab, m, k, s, seed, mode=mode, f="invsqrt", cond_max=cond_max,
                              lsqr_tol=lsqr_tol, lsqr_iters=lsqr_iters)
    return solve(A2, Ab, m, k, s, seed, mode=mode, f="invsqrt", lsqr_tol=lsqr_tol, lsqr_iters=lsqr_iters,
                 keep=keep)

"""Krylov bases: Algorithm 1 (sketched Gram-Schmidt, PAPER.md l.61-100,
§2.1.1), Algorithm 2 (truncated orthogonalization, l.102-130, §2.1.2) and
the Arnoldi decomposition (Eq. (2), l.38-48).

Algorithm 2 as printed (l.118-127):
    v_1 <- b / ||b||_2
    for i = 2 .. m+1:
        w_i <- A v_{i-1}
        for j = max{1, i-k} .. i-1:
            h_{j,i-1} <- v_j^T w_i
            w_i <- w_i - h_{j,i} v_i           (typo, G-1: read h_{j,i-1} v_j)
        h_{i,i-1} <- ||w||_2                   (read ||w_i||_2)
        v_i <- w_i / ||w_i||_2
Reading G-1 restores the evident orthogonalization.  ``variant="mgs"`` is the
literal sequential loop; ``variant="cgs"`` computes all k window coefficients
from the un-updated w_i first (one-pass classical GS, equal in exact
arithmetic because the window is orthonormal, G-2).  Breakdown (G-5): stop
when h_{i,i-1} <= 1e-14 ||A||_inf; then m_eff = i-1 and K_{m_eff} is an
invariant subspace.

Indices: code is 0-based, column c of V is the paper's v_{c+1}; H is the
(m+1) x m matrix underline-H_m with H[c', c] = h_{c'+1, c+1}.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np


def _norm_inf(A):
    return float(abs(A).sum(axis=1).max())


def truncated_arnoldi(A, b, m: int, k: int, variant: str = "mgs",
                      breakdown_tol: float = 1e-14, V_out=None):
    """Algorithm 2.  Returns dict(V, H, gamma=||b||_2, m_eff, breakdown):
    V is n x (m+1) and H (m+1) x m without breakdown; on breakdown at step
    i, m_eff = i-1, V = [v_1..v_{m_eff}] and H is (m_eff+1) x m_eff.
    V_out: optional zero-filled n x (m+1) array to hold V (e.g. a
    column-major np.memmap when V exceeds host memory, c5); same arithmetic."""
    n = b.shape[0]
    if k < 1 or m < 1:
        raise ValueError("need k >= 1, m >= 1")
    gamma = float(np.linalg.norm(b))
    V = np.zeros((n, m + 1)) if V_out is None else V_out
    H = np.zeros((m + 1, m))
    V[:, 0] = b / gamma                                   # l.118
    thresh = breakdown_tol * _norm_inf(A)
    for i in range(2, m + 2):                             # l.119, paper index i
        c = i - 1                                          # 0-based new column
        w = A @ V[:, c - 1]                                # l.120
        js = range(max(1, i - k), i)                       # l.121, paper j
        if variant == "mgs":
            for j in js:
                H[j - 1, c - 1] = V[:, j - 1] @ w          # l.122
                w = w - H[j - 1, c - 1] * V[:, j - 1]      # l.123 (G-1)
        elif variant == "cgs":
            W = V[:, [j - 1 for j in js]]
            hc = W.T @ w
            for t, j in enumerate(js):
                H[j - 1, c - 1] = hc[t]
            w = w - W @ hc
        else:
            raise ValueError(variant)
        hn = float(np.linalg.norm(w))                      # l.125
        H[c, c - 1] = hn
        if hn <= thresh:                                   # G-5
            # K_{i-1} is A-invariant: m_eff = i-1; V keeps v_1..v_{i-1} only
            m_eff = c
            return dict(V=V[:, :m_eff], H=H[: m_eff + 1, :m_eff],
                        gamma=gamma, m_eff=m_eff, breakdown=True)
        V[:, c] = w / hn                                   # l.126
    return dict(V=V, H=H, gamma=gamma, m_eff=m, breakdown=False)


def arnoldi(A, b, m: int, breakdown_tol: float = 1e-14):
    """Arnoldi decomposition Eq. (2): A U_m = U_{m+1} K_m (underline), U
    orthonormal; modified Gram-Schmidt with one full reorthogonalization
    pass (the 'exact' reference of PAPER.md l.358)."""
    n = b.shape[0]
    gamma = float(np.linalg.norm(b))
    U = np.zeros((n, m + 1))
    K = np.zeros((m + 1, m))
    U[:, 0] = b / gamma
    thresh = breakdown_tol * _norm_inf(A)
    for c in range(1, m + 1):
        w = A @ U[:, c - 1]
        for _pass in range(2):
            for j in range(c):
                hj = U[:, j] @ w
                K[j, c - 1] += hj
                w = w - hj * U[:, j]
        hn = float(np.linalg.norm(w))
        K[c, c - 1] = hn
        if hn <= thresh:
            return dict(V=U[:, :c], H=K[: c + 1, :c], gamma=gamma,
                        m_eff=c, breakdown=True)
        U[:, c] = w / hn
    return dict(V=U, H=K, gamma=gamma, m_eff=m, breakdown=False)


def sketched_gs(A, b, m: int, theta, breakdown_tol: float = 1e-14):
    """Algorithm 1 (after Balabanov & Grigori), literally:

        w_1 <- b;  p_1 <- Theta w_1;  r_11 <- ||p_1||;  s_1 <- p_1 / r_11;
        v_1 <- w_1 / r_11
        for i = 2 .. m+1:
            w_i <- A v_{i-1}                          (l.89)
            p_i <- Theta w_i                          (l.90)
            r_i <- S_{i-1}^T p_i;  R(1:i-1, i) <- r_i  (l.91)
            s_i <- p_i - S_{i-1} r_i                  (l.92)
            r_ii <- ||s_i||                           (l.93)
            s_i <- s_i / r_ii;  S_i <- [S_{i-1} s_i]  (l.94)
            v_i <- (w_i - V_{i-1} r_i) / r_ii         (l.95)
        underline-H_m <- R(:, 2:m+1)                  (l.97)

    theta: an object with .apply(x) = Theta x (oracle.srht.SRHT).
    Breakdown (reading G-5 applied to r_ii, the sketched norm of the new
    direction): stop when r_ii <= 1e-14 ||A||_inf ||Theta v_{i-1}||-scale,
    i.e. r_ii <= 1e-14 ||A||_inf (S is orthonormal, so ||Theta v_j|| = 1).
    Returns dict(V, H, S, R, gamma=r_11, m_eff, breakdown)."""
    n = b.shape[0]
    V = np.zeros((n, m + 1))
    R = np.zeros((m + 1, m + 1))
    p1 = theta.apply(b)
    s = p1.shape[0]
    S = np.zeros((s, m + 1))
    r11 = float(np.linalg.norm(p1))                      # l.86
    R[0, 0] = r11
    S[:, 0] = p1 / r11                                    # l.87
    V[:, 0] = b / r11                                     # l.88
    thresh = breakdown_tol * _norm_inf(A)
    for i in range(2, m + 2):                             # l.89 (paper index)
        c = i - 1
        w = A @ V[:, c - 1]
        p = theta.apply(w)
        r = S[:, :c].T @ p                                # l.91
        R[:c, c] = r
        sv = p - S[:, :c] @ r                             # l.92
        rii = float(np.linalg.norm(sv))                   # l.93
        R[c, c] = rii
        if rii <= thresh:
            m_eff = c
            return dict(V=V[:, :m_eff], H=R[: m_eff + 1, 1: m_eff + 1], S=S[:, :m_eff],
                        R=R[: m_eff + 1, : m_eff + 1], gamma=r11, m_eff=m_eff, breakdown=True)
        S[:, c] = sv / rii                                # l.94
        V[:, c] = (w - V[:, :c] @ r) / rii                # l.95
    return dict(V=V, H=R[:, 1:], S=S, R=R, gamma=r11, m_eff=m, breakdown=False)


def cond1_upper(R):
    """||R||_1 ||R^{-1}||_1 of an upper-triangular R (exact, by triangular
    solves): the conditioning measure of the sketched basis (reading R-5)."""
    from .lsq import solve_upper
    m = R.shape[0]
    Ri = solve_upper(R, np.eye(m))
    return float(np.abs(R).sum(axis=0).max() * np.abs(Ri).sum(axis=0).max())


def whitened_basis(A, b, m: int, k: int, theta, cond_max: float = 1000.0,
                   breakdown_tol: float = 1e-14):
    """Algorithm 2 with whitening (§5.1.3 l.395), literally:

    run Algorithm 2 (truncated orthogonalisation, MGS window as printed); after
    each new basis vector (V_i, i = 2, 3, ...) form the sketch Theta V_i and
    its QR factor R_i (Householder, R_jj >= 0); the first time the
    conditioning of Theta V_i exceeds cond_max (l.395: 1000; measured as
    ||R_i||_1 ||R_i^{-1}||_1, reading R-5), whiten:
        V_i <- V_i R_i^{-1},   underline-H_{i-1} <- R_i underline-H_{i-1} R_{i-1}^{-1}
    and "continue the construction of the basis as in Algorithm 1, using the
    same sketch matrix Theta" (l.106) up to V_{m+1}; then V_{m+1} satisfies
    the Arnoldi-like relation Eq. (3) with the sketch S = Theta V orthonormal
    from column i on.  gamma = ||b||_2 R_11 (V^+ b = gamma e_1).
    Returns dict(V, H, gamma, m_eff, breakdown, whitened_at (i or 0))."""
    from .lsq import householder_qr, solve_upper
    n = b.shape[0]
    thresh = breakdown_tol * _norm_inf(A)
    gamma = float(np.linalg.norm(b))
    V = np.zeros((n, m + 1))
    H = np.zeros((m + 1, m))
    V[:, 0] = b / gamma
    i_w = 0
    for i in range(2, m + 2):                                    # Algorithm 2 steps
        c = i - 1
        w = A @ V[:, c - 1]
        for j in range(max(1, i - k), i):
            H[j - 1, c - 1] = V[:, j - 1] @ w
            w = w - H[j - 1, c - 1] * V[:, j - 1]
        hn = float(np.linalg.norm(w))
        H[c, c - 1] = hn
        if hn <= thresh:
            return dict(V=V[:, :c], H=H[: c + 1, :c], gamma=gamma, m_eff=c, breakdown=True,
                        whitened_at=0)
        V[:, c] = w / hn
        if c + 1 == m + 1:
            break                                                # V_{m+1} complete without whitening
        R, _ = householder_qr(theta.apply(V[:, : c + 1]))       # Theta V_i = Q_i R_i, i = c+1
        if cond1_upper(R) > cond_max:
            i_w = c + 1
            V[:, :i_w] = V[:, :i_w] @ solve_upper(R, np.eye(i_w))
            Hs = H[:i_w, : i_w - 1]
            H[:i_w, : i_w - 1] = R @ Hs @ solve_upper(R[: i_w - 1, : i_w - 1], np.eye(i_w - 1))
            gamma = gamma * float(R[0, 0])
            break
    if i_w == 0:
        return dict(V=V, H=H, gamma=gamma, m_eff=m, breakdown=False, whitened_at=0)
    # Algorithm 1 from column i_w on (l.89-95), S = Theta V (orthonormal)
    S = np.zeros((theta.s, m + 1))
    S[:, :i_w] = theta.apply(V[:, :i_w])
    for i in range(i_w + 1, m + 2):
        c = i - 1
        w = A @ V[:, c - 1]
        p = theta.apply(w)
        r = S[:, :c].T @ p
        sv = p - S[:, :c] @ r
        rii = float(np.linalg.norm(sv))
        H[:c, c - 1] = r
        H[c, c - 1] = rii
        if rii <= thresh:
            return dict(V=V[:, :c], H=H[: c + 1, :c], gamma=gamma, m_eff=c, breakdown=True,
                        whitened_at=i_w)
        S[:, c] = sv / rii
        V[:, c] = (w - V[:, :c] @ r) / rii
    return dict(V=V, H=H, gamma=gamma, m_eff=m, breakdown=False, whitened_at=i_w)

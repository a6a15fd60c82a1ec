"""Row-partitioned model of the multi-GPU decomposition (TEST INFRASTRUCTURE).

Each torch.distributed rank (gloo, CPU) runs, in numpy, exactly the data
movement libfab.so's comm.cu performs on several GPUs:

  * rows [r0, r1) of A, b, V per rank, from the product's partition plan
    (paper_2212_12758_b200.dist);
  * C1 halo: the first / last `hal` rows of w_hat_{i-1} go to ranks p-1 /
    p+1 (send/recv), so the local SpMV sees rows [r0-hal, r1+hal);
  * C2: ONE allreduce of the k+1 step scalars (window dots + the lagged
    norm of the previous column, reading G-4) per Krylov step;
  * C3: sketch partials of the rank's rows on GLOBALLY aligned 4096-row
    tiles (reading R-1; blocks are not tile aligned), one allreduce;
  * C4: LSQR on the distributed basis, with the m+1 pass scalars
    (g = W^T t and ||t||^2) allreduced.

The single-process oracle is the reference the tests compare against.
"""
import math

import numpy as np
import torch
import torch.distributed as dist

from oracle import lsq, matfun
from oracle.srht import SRHT, fwht

T = 4096


def allreduce(a):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def halo_exchange(x, hal, rank, P):
    """[rows r0-hal .. r0-1 | x | rows r1 .. r1+hal-1] (zeros off the ends)."""
    lo = torch.zeros(hal, dtype=torch.float64)
    hi = torch.zeros(hal, dtype=torch.float64)
    xt = torch.from_numpy(np.ascontiguousarray(x))
    ops = []
    if rank > 0:
        ops += [dist.P2POp(dist.isend, xt[:hal].clone(), rank - 1), dist.P2POp(dist.irecv, lo, rank - 1)]
    if rank + 1 < P:
        ops += [dist.P2POp(dist.isend, xt[-hal:].clone(), rank + 1), dist.P2POp(dist.irecv, hi, rank + 1)]
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return np.concatenate([lo.numpy(), x, hi.numpy()])


def gather_x(x, cuts, rank, P):
    """C1 for CSR: all-gather-v of the ranks' rows into a global vector."""
    parts = [torch.zeros(int(cuts[q + 1] - cuts[q]), dtype=torch.float64) for q in range(P)]
    xt = torch.from_numpy(np.ascontiguousarray(x))
    ops = []
    for q in range(P):
        if q != rank:
            ops += [dist.P2POp(dist.isend, xt.clone(), q), dist.P2POp(dist.irecv, parts[q], q)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    parts[rank] = xt
    return torch.cat(parts).numpy()


def local_sketch_partial(x_loc, r0, th):
    """sum over the global tiles touched by rows [r0, r0+len): the pruned
    FWHT partial of R-1, for the s sampled rows (unscaled)."""
    n_loc = len(x_loc)
    out = np.zeros(th.s)
    hi = th.rows >> 12
    lo = th.rows & (T - 1)
    for tile in range(r0 >> 12, ((r0 + n_loc - 1) >> 12) + 1):
        g0 = tile * T
        v = np.zeros(T)
        a, b = max(g0, r0), min(g0 + T, r0 + n_loc)
        v[a - g0:b - g0] = x_loc[a - r0:b - r0] * th.signs[a:b]
        y = fwht(v)
        par = np.array([bin(int(h) & tile).count("1") & 1 for h in hi])
        out += np.where(par == 1, -1.0, 1.0) * y[lo]
    return out


def rank_solve(rank, P, A, b, cuts, hal, m, k, s, seed, f, alpha, sigma, lsqr_iters, square=False):
    """One rank of the row-partitioned Algorithm 4 (Blendenpik, fixed L).
    hal = halo rows (stencil) or None (CSR: gathered x).  square: the
    operator is A^2 applied as A (A w) with a C1 exchange before each of the
    two products, and the start vector is A b (FAB_FLAG_SQUARE, sign(A) b by
    l.406).  Returns (f_m rows, H, SV, y) of this rank (H, SV, y replicated)."""
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    n_loc = r1 - r0
    n = A.shape[0]
    import scipy.sparse as sp
    if hal is None:
        # CSR: x is gathered to global length every step (C1, all-gather-v)
        A_ext = A[r0:r1].tocsr()
    else:
        # stencil: local rows of A restricted to columns [r0-hal, r1+hal)
        A_loc = A[r0:r1].tocoo()
        lo_col = r0 - hal
        assert A_loc.col.min() >= lo_col and A_loc.col.max() < r1 + hal, "halo too narrow"
        A_ext = sp.csr_matrix((A_loc.data, (A_loc.row, A_loc.col - lo_col)), shape=(n_loc, n_loc + 2 * hal))

    def spmv(x):                                                  # C1 + one local product
        if hal is None:
            xe = gather_x(x, cuts, rank, P)
        else:
            xe = halo_exchange(x, hal, rank, P) if P > 1 else np.concatenate([np.zeros(hal), x, np.zeros(hal)])
        return A_ext @ xe

    W = np.zeros((n_loc, m + 1))
    W[:, 0] = spmv(b[r0:r1]) if square else b[r0:r1]
    H = np.zeros((m + 1, m))
    beta = np.zeros(m + 1)
    nu_loc = W[:, 0] @ W[:, 0]
    for c in range(1, m + 1):
        x = W[:, c - 1]
        z = spmv(spmv(x)) if square else spmv(x)                   # (K0 +) K1
        js = list(range(max(0, c - k), c))
        red = allreduce(np.array([W[:, j] @ z for j in js] + [nu_loc]))   # C2: k+1 scalars
        beta[c - 1] = math.sqrt(red[-1])
        if c >= 2:
            H[c - 1, c - 2] = beta[c - 1]
        w = z / beta[c - 1]
        for t, j in enumerate(js):
            h = red[t] / (beta[j] * beta[c - 1])
            H[j, c - 1] = h
            w = w - (h / beta[j]) * W[:, j]
        W[:, c] = w
        nu_loc = w @ w
    beta[m] = math.sqrt(allreduce(np.array([nu_loc]))[0])
    H[m, m - 1] = beta[m]
    Vloc = W / beta                                               # normalised v_j (local rows)

    th = SRHT(n, s, seed)
    SV = np.stack([local_sketch_partial(W[:, j], r0, th) for j in range(m + 1)], axis=1)
    SV = allreduce(SV) / (math.sqrt(s) * beta)                    # C3

    # Blendenpik-LSQR on the distributed basis (C4: allreduced pass scalars)
    R, _ = lsq.householder_qr(SV[:, :m])
    Vm, c_rhs = Vloc[:, :m], Vloc[:, m]

    def gnorm(u):
        return math.sqrt(allreduce(np.array([u @ u]))[0])

    def rmatvec(u):                                              # R^-T V^T u
        return lsq.solve_upper_transposed(R, allreduce(Vm.T @ u))

    def matvec(p):
        return Vm @ lsq.solve_upper(R, p)

    zc = np.zeros(m)
    bt = gnorm(c_rhs)
    u = c_rhs / bt
    v = rmatvec(u)
    al = float(np.linalg.norm(v))
    v = v / al
    wv = v.copy()
    phibar, rhobar = bt, al
    for _ in range(lsqr_iters):
        u = matvec(v) - al * u
        bt = gnorm(u)
        u = u / bt
        v = rmatvec(u) - bt * v
        al = float(np.linalg.norm(v))
        v = v / al
        rho = math.hypot(rhobar, bt)
        cs, sn = rhobar / rho, bt / rho
        theta = sn * al
        rhobar = -cs * al
        phi = cs * phibar
        phibar = sn * phibar
        zc = zc + (phi / rho) * wv
        wv = v - (theta / rho) * wv
    y = lsq.solve_upper(R, zc)
    C = H[:m, :m].copy()
    C[:, m - 1] += H[m, m - 1] * y                                # Eq. (6)
    cvec = matfun.f_e1(f, C, alpha, sigma)
    fm_loc = beta[0] * (Vm @ cvec)
    return fm_loc, H, SV, y

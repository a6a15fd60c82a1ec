"""Seeded synthetic inputs for the f(A)b hot path (BASELINE.json configs c1..c5).

This module is shared by the oracle (``oracle/``), the tests and ``bench.py``.
It holds NONE of the method's arithmetic (no Krylov step, no sketch, no least
squares, no matrix function): it only assembles the operator A and the vector
b that the paper's method is applied to.  Every input is a deterministic
function of its seed (numpy PCG64 ``default_rng``).

Workload recipes (readings G-20,
G-23, G-25, G-26, G-27):

* c1/c2: 2D convection-diffusion -D*Lap(u) + v.grad(u), D = 1, v = (10, 10),
  first-order upwind, homogeneous Dirichlet, g x g interior grid,
  h = 1/(g+1), lexicographic order (x fastest); scaled so ||A||_inf = 1e3.
  Stand-in for the paper's conv-diff experiments.
* c3: the 3D analogue (7-point, v = (10,10,10)), unscaled, g = 256.
  Stand-in for the 3D Laplacian / conv-diff experiments (PAPER.md
  l.415-429, l.434-442).
* c4: Chung-Lu power-law graph adjacency (exponent 2.5, mean degree 12),
  divided by a Lanczos estimate of lambda_max.  Stand-in for the graph
  experiments (p2p-Gnutella08, wiki-Vote) whose
  datasets are not available here.
* c5: nonsymmetric random sparse, 16 distinct uniform columns per row,
  values N(0,1)/4, diagonal shifted by -5.  Stand-in for the nonnormal
  examples.

The paper's own experiments that need no dataset:

* e1: the variable-coefficient convection-diffusion operator of PAPER.md
  l.366-374 (Pe = 200, D1 = 1000 on [1/4,3/4]^2 else 1, D2 = D1/2,
  v = (x+y, x-y), skew-symmetric convection form) on a 352 x 352 grid,
  b = sin(pi x) sin(pi y) normalized, f = exp(-t A) with t = 1e3/||A||_inf
  (reading G-30).  CSR (variable coefficients).
* e4: stand-in for the sign-function example (bfw782a, not
  available): nonsymmetric random sparse as c5 but with the diagonal shift
  +-5 by a seeded Rademacher sign per row (spectrum in both half planes),
  b a random unit vector, f = sign via (A^2)^{-1/2} (A b).
* e5: the 3D Laplacian of PAPER.md l.417-421, T_N (x) I (x) I + I (x) T_N (x) I
  + I (x) I (x) T_N, T_N = tridiag(-1, 2, -1) (G-28), N = 80, f = invsqrt,
  b a random unit vector, sketch s = floor(1.05 m) (l.421).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = ["Problem", "make", "CONFIGS", "stencil_coeffs", "stencil_csr", "stencil_row",
           "chung_lu", "random_sparse", "gaussian_b"]

# (center, x-, x+, y-, y+, z-, z+)
COEFF_NAMES = ("center", "xm", "xp", "ym", "yp", "zm", "zp")


@dataclasses.dataclass
class Problem:
    name: str
    n: int
    kind: str                      # "stencil" | "csr"
    b: np.ndarray
    f: str                         # "exp" | "sqrt" | "invsqrt" | "sign"
    alpha: float
    sigma: float
    m: int
    k: int
    s: int
    sketch_seed: int
    norm_inf: float
    dims: tuple = (0, 0, 0)        # stencil grid (gx, gy, gz); gz = 1 in 2D
    coeffs: tuple = ()             # 7 stencil coefficients (already scaled)
    _csr: Optional[tuple] = None   # (indptr int64, indices int32, data f64)
    meta: dict = dataclasses.field(default_factory=dict)

    def csr(self):
        """(indptr, indices, data) of A; assembled lazily for stencils."""
        if self._csr is None:
            assert self.kind == "stencil"
            self._csr = stencil_csr(self.dims, self.coeffs)
        return self._csr

    def scipy(self):
        import scipy.sparse as sp
        ip, ix, dv = self.csr()
        return sp.csr_matrix((dv, ix, ip), shape=(self.n, self.n))


# ----------------------------------------------------------------------------
# stencils
# ----------------------------------------------------------------------------
def stencil_coeffs(dim: int, g: int, D: float = 1.0, v: float = 10.0,
                   scale_to: Optional[float] = None):
    """Upwind convection-diffusion coefficients (G-20).

    Returns (coeffs, norm_inf) with coeffs = (center, x-, x+, y-, y+, z-, z+)
    (z entries zero in 2D).  Diffusion: 2*dim*D/h^2 on the centre and -D/h^2
    on every neighbour; convection v>0 by backward differences: +v/h on the
    centre and -v/h on the upwind (minus) neighbour.
    """
    h = 1.0 / (g + 1)
    dd = D / (h * h)
    vh = v / h
    center = 2 * dim * dd + dim * vh
    minus = -dd - vh
    plus = -dd
    c = [center, minus, plus, minus, plus, 0.0, 0.0]
    if dim == 3:
        c[5], c[6] = minus, plus
    norm_inf = abs(center) + dim * (abs(minus) + abs(plus))
    if scale_to is not None:
        sc = scale_to / norm_inf
        c = [x * sc for x in c]
        norm_inf = abs(c[0]) + dim * (abs(c[1]) + abs(c[2]))
    return tuple(float(x) for x in c), float(norm_inf)


def stencil_csr(dims, coeffs):
    """Assemble the CSR of the constant-coefficient stencil (Dirichlet BC).

    Row r = x + gx*(y + gy*z); columns sorted ascending per row.
    """
    gx, gy, gz = dims
    n = gx * gy * gz
    r = np.arange(n, dtype=np.int64)
    x = r % gx
    y = (r // gx) % gy
    z = r // (gx * gy)
    c0, cxm, cxp, cym, cyp, czm, czp = coeffs
    # ascending column order: z-, y-, x-, centre, x+, y+, z+
    slots = [
        (-gx * gy, czm, z > 0),
        (-gx, cym, y > 0),
        (-1, cxm, x > 0),
        (0, c0, np.ones(n, dtype=bool)),
        (1, cxp, x < gx - 1),
        (gx, cyp, y < gy - 1),
        (gx * gy, czp, z < gz - 1),
    ]
    # in 2D (gz == 1) the z masks are all False, so those slots drop out
    cols = np.stack([r + off for off, _, _ in slots], axis=1)
    vals = np.stack([np.full(n, cv) for _, cv, _ in slots], axis=1)
    mask = np.stack([np.broadcast_to(mk, (n,)) for _, _, mk in slots], axis=1)
    counts = mask.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    indices = cols[mask].astype(np.int32)
    data = vals[mask].astype(np.float64)
    return indptr, indices, data


def stencil_row(dims, coeffs, r):
    """(columns, values) of row r of the stencil operator (ascending
    columns, Dirichlet boundary): the same operator as stencil_csr, one row
    at a time for full-size spot checks."""
    gx, gy, gz = dims
    x, y, z = r % gx, (r // gx) % gy, r // (gx * gy)
    c0, cxm, cxp, cym, cyp, czm, czp = coeffs
    ent = [(-gx * gy, czm, z > 0), (-gx, cym, y > 0), (-1, cxm, x > 0), (0, c0, True),
           (1, cxp, x < gx - 1), (gx, cyp, y < gy - 1), (gx * gy, czp, z < gz - 1)]
    cols = [r + off for off, _, ok in ent if ok]
    vals = [v for _, v, ok in ent if ok]
    return np.asarray(cols, dtype=np.int64), np.asarray(vals, dtype=np.float64)


# ----------------------------------------------------------------------------
# graphs / random sparse
# ----------------------------------------------------------------------------
def _csr_from_coo(n, rows, cols, vals):
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    counts = np.bincount(rows, minlength=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return indptr, cols.astype(np.int32), vals.astype(np.float64)


def chung_lu(n: int, seed: int, mean_deg: float = 12.0, beta: float = 2.5):
    """Symmetric 0/1 Chung-Lu adjacency (G-25).  Returns CSR with data = 1."""
    rng = np.random.default_rng(seed)
    w = (np.arange(n, dtype=np.float64) + 1.0) ** (-1.0 / (beta - 1.0))
    w *= mean_deg * n / w.sum()
    cap = math.sqrt(w.sum())
    w = np.minimum(w, cap)
    w *= mean_deg * n / w.sum()
    total = w.sum()
    n_pairs = int(rng.poisson(total / 2.0))
    cdf = np.cumsum(w / total)
    cdf[-1] = 1.0
    src = np.minimum(np.searchsorted(cdf, rng.random(n_pairs), side="right"), n - 1)
    dst = np.minimum(np.searchsorted(cdf, rng.random(n_pairs), side="right"), n - 1)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    keys = np.concatenate([src * n + dst, dst * n + src])
    keys = np.unique(keys)
    rows = keys // n
    cols = keys % n
    return _csr_from_coo(n, rows, cols, np.ones(len(keys)))


def lanczos_lambda_max(indptr, indices, data, n, steps=64):
    """Top Ritz value of a fully reorthogonalized Lanczos run from the
    all-ones vector: the lambda_max estimate used to scale c4 (G-25).
    Input preparation only (a scaling constant of A), not the method."""
    import scipy.sparse as sp
    from scipy.linalg import eigh_tridiagonal
    A = sp.csr_matrix((data, indices, indptr), shape=(n, n))
    steps = min(steps, n)
    Q = np.zeros((steps + 1, n))
    q = np.ones(n) / math.sqrt(n)
    Q[0] = q
    al, be = [], []
    for j in range(steps):
        w = A @ Q[j]
        a = float(Q[j] @ w)
        w -= Q[: j + 1].T @ (Q[: j + 1] @ w)
        w -= Q[: j + 1].T @ (Q[: j + 1] @ w)
        bnorm = float(np.linalg.norm(w))
        al.append(a)
        if bnorm < 1e-12 or j == steps - 1:
            break
        be.append(bnorm)
        Q[j + 1] = w / bnorm
    ev = eigh_tridiagonal(np.array(al), np.array(be[: len(al) - 1]), eigvals_only=True)
    return float(ev[-1])


def random_sparse(n: int, seed: int, per_row: int = 16, shift=-5.0,
                  scale: float = 0.25):
    """Nonsymmetric random sparse matrix (G-26): per row `per_row` distinct
    uniform columns with N(0,1)*scale values, plus `shift` on the diagonal
    (merged into an existing diagonal entry when one was drawn).  `shift`
    is a scalar or a per-row array (e4)."""
    rng = np.random.default_rng(seed)
    per_row = min(per_row, n)
    cols = rng.integers(0, n, size=(n, per_row), dtype=np.int64)
    while True:
        cols.sort(axis=1)
        dup = np.zeros_like(cols, dtype=bool)
        dup[:, 1:] = cols[:, 1:] == cols[:, :-1]
        nd = int(dup.sum())
        if nd == 0:
            break
        cols[dup] = rng.integers(0, n, size=nd, dtype=np.int64)
    vals = rng.standard_normal((n, per_row)) * scale
    r = np.arange(n, dtype=np.int64)
    is_diag = cols == r[:, None]
    has_diag = is_diag.any(axis=1)
    shift_r = np.broadcast_to(np.asarray(shift, dtype=np.float64), (n,))
    vals[is_diag] += np.broadcast_to(shift_r[:, None], vals.shape)[is_diag]
    extra_col = np.where(has_diag, n, r)            # n = sentinel (dropped)
    extra_val = np.where(has_diag, 0.0, shift_r)
    cols = np.concatenate([cols, extra_col[:, None]], axis=1)
    vals = np.concatenate([vals, extra_val[:, None]], axis=1)
    order = np.argsort(cols, axis=1, kind="stable")
    cols = np.take_along_axis(cols, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    mask = cols < n
    counts = mask.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return indptr, cols[mask].astype(np.int32), vals[mask].astype(np.float64)


def convdiff_var(g: int, pe: float = 200.0):
    """CSR of the variable-coefficient convection-diffusion operator of
    PAPER.md l.366-374 on the unit square, g x g interior points, h = 1/(g+1),
    homogeneous Dirichlet, x fastest:
      L[u] = -(D1 u_x)_x - (D2 u_y)_y + Pe (1/2 (v1 u_x + v2 u_y)
             + 1/2 ((v1 u)_x + (v2 u)_y)),
      D1 = 1000 on [1/4, 3/4]^2 else 1, D2 = D1/2, v1 = x+y, v2 = x-y.
    Second-order finite differences (reading G-31): the diffusion flux with
    D at the cell faces (x +- h/2), both convection terms by central
    differences."""
    h = 1.0 / (g + 1)
    n = g * g
    r = np.arange(n, dtype=np.int64)
    ix = r % g
    iy = r // g
    x = (ix + 1) * h
    y = (iy + 1) * h

    def d1(px, py):
        inside = (px >= 0.25) & (px <= 0.75) & (py >= 0.25) & (py <= 0.75)
        return np.where(inside, 1000.0, 1.0)

    dxm, dxp = d1(x - h / 2, y), d1(x + h / 2, y)
    dym, dyp = 0.5 * d1(x, y - h / 2), 0.5 * d1(x, y + h / 2)
    v1 = lambda px, py: px + py          # noqa: E731
    v2 = lambda px, py: px - py          # noqa: E731
    h2, c2 = h * h, pe / (4.0 * h)
    # u_x ~ (u_{i+1} - u_{i-1}) / 2h;  (v1 u)_x ~ (v1_{i+1} u_{i+1} - v1_{i-1} u_{i-1}) / 2h
    cxm = -dxm / h2 - c2 * (v1(x, y) + v1(x - h, y))
    cxp = -dxp / h2 + c2 * (v1(x, y) + v1(x + h, y))
    cym = -dym / h2 - c2 * (v2(x, y) + v2(x, y - h))
    cyp = -dyp / h2 + c2 * (v2(x, y) + v2(x, y + h))
    cc = (dxm + dxp + dym + dyp) / h2
    slots = [(-g, cym, iy > 0), (-1, cxm, ix > 0), (0, cc, np.ones(n, dtype=bool)),
             (1, cxp, ix < g - 1), (g, cyp, iy < g - 1)]
    cols = np.stack([r + off for off, _, _ in slots], axis=1)
    vals = np.stack([v for _, v, _ in slots], axis=1)
    mask = np.stack([mk for _, _, mk in slots], axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(axis=1), out=indptr[1:])
    return indptr, cols[mask].astype(np.int32), vals[mask].astype(np.float64)


def gaussian_b(n: int, seed: int, normalize: bool = False):
    b = np.random.default_rng(seed).standard_normal(n)
    if normalize:
        b /= np.linalg.norm(b)
    return b


def csr_norm_inf(indptr, data):
    rs = np.add.reduceat(np.abs(data), indptr[:-1]) if len(data) else np.zeros(len(indptr) - 1)
    empty = indptr[1:] == indptr[:-1]
    rs[empty] = 0.0
    return float(rs.max()) if len(rs) else 0.0


# ----------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------
CONFIGS = {
    # name: defaults (full size)
    "c1": dict(g=100, m=40, k=2, s=80),
    "c2": dict(g=1000, m=100, k=2, s=200),
    "c3": dict(g=256, m=200, k=4, s=400),
    "c4": dict(n=1 << 22, m=150, k=2, s=300),
    "c5": dict(n=1 << 25, m=300, k=2, s=600),
    # the paper's dataset-free experiments (defaults: one point of the m sweep)
    "e1": dict(g=352, m=60, k=2, s=120),
    "e4": dict(n=1 << 20, m=40, k=2, s=80),
    "e5": dict(g=80, m=100, k=2, s=None),
}


def make(name: str, **over) -> Problem:
    """Build config `name` ("c1".."c5"); keyword overrides shrink it for tests
    (g= grid side, n= size, m=, k=, s=; unscaled=True for the c2 stress
    variant of G-23)."""
    if name not in CONFIGS:
        raise KeyError(name)
    p = dict(CONFIGS[name])
    p.update(over)
    idx = int(name[1]) + (10 if name[0] == "e" else 0)
    mseed, bseed, sseed = 1000 + idx, 2000 + idx, 3000 + idx
    m, k, s = p["m"], p["k"], p["s"]
    if name == "e5" and s is None:
        s = int(math.floor(1.05 * m))               # l.421
    if name == "e1":
        g = p["g"]
        ip, ix, dv = convdiff_var(g)
        ninf = csr_norm_inf(ip, dv)
        t = 1e3 / ninf                               # G-30
        hh = 1.0 / (g + 1)
        xs = np.sin(np.pi * hh * np.arange(1, g + 1))
        b = np.outer(xs, xs).ravel()                 # sin(pi x) sin(pi y), x fastest (symmetric)
        b /= np.linalg.norm(b)
        return Problem(name, g * g, "csr", b, "exp", -t, 0.0, m, k, s, sseed, ninf, _csr=(ip, ix, dv),
                       meta=dict(g=g, t=t, nnz=int(ip[-1])))
    if name == "e4":
        n = p["n"]
        sg = np.where(np.random.default_rng(mseed + 500).random(n) < 0.5, -5.0, 5.0)
        ip, ix, dv = random_sparse(n, mseed, shift=sg)
        b = gaussian_b(n, bseed, normalize=True)
        return Problem(name, n, "csr", b, "sign", 1.0, 0.0, m, k, s, sseed, csr_norm_inf(ip, dv),
                       _csr=(ip, ix, dv), meta=dict(nnz=int(ip[-1])))
    if name == "e5":
        g = p["g"]
        c = (6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0)
        n = g ** 3
        b = gaussian_b(n, bseed, normalize=True)
        return Problem(name, n, "stencil", b, "invsqrt", 1.0, 0.0, m, k, s, sseed, 12.0,
                       dims=(g, g, g), coeffs=c, meta=dict(g=g, dim=3))
    if name in ("c1", "c2"):
        g = p["g"]
        scale_to = None if p.get("unscaled") else 1e3
        coeffs, ninf = stencil_coeffs(2, g, scale_to=scale_to)
        n = g * g
        b = gaussian_b(n, bseed, normalize=(name == "c1"))
        alpha = -1.0 if name == "c1" else -1e-3
        return Problem(name, n, "stencil", b, "exp", alpha, 0.0, m, k, s, sseed,
                       ninf, dims=(g, g, 1), coeffs=coeffs,
                       meta=dict(g=g, dim=2, scaled=scale_to is not None))
    if name == "c3":
        g = p["g"]
        coeffs, ninf = stencil_coeffs(3, g)
        n = g ** 3
        b = gaussian_b(n, bseed)
        return Problem(name, n, "stencil", b, "sqrt", 1.0, 1e-2 * ninf, m, k, s,
                       sseed, ninf, dims=(g, g, g), coeffs=coeffs,
                       meta=dict(g=g, dim=3))
    if name == "c4":
        n = p["n"]
        ip, ix, dv = chung_lu(n, mseed)
        lam = lanczos_lambda_max(ip, ix, dv, n)
        dv = dv / lam
        rng = np.random.default_rng(bseed)
        b = np.where(rng.random(n) < 0.5, -1.0, 1.0) / math.sqrt(n)
        return Problem(name, n, "csr", b, "exp", 1.0, 0.0, m, k, s, sseed,
                       csr_norm_inf(ip, dv), _csr=(ip, ix, dv),
                       meta=dict(lambda_hat=lam, nnz=int(ip[-1]),
                                 max_deg=int(np.diff(ip).max())))
    if name == "c5":
        n = p["n"]
        ip, ix, dv = random_sparse(n, mseed)
        b = gaussian_b(n, bseed)
        return Problem(name, n, "csr", b, "invsqrt", -1.0, 0.0, m, k, s, sseed,
                       csr_norm_inf(ip, dv), _csr=(ip, ix, dv),
                       meta=dict(nnz=int(ip[-1])))
    raise KeyError(name)

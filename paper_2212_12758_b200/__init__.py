"""B200-native randomized Krylov f(A)b (arXiv 2212.12758): Python binding.

Thin wrapper over the C ABI in include/fab.h (libfab.so, sm_100a).  PyTorch
is used only for device memory and streams; every step of the path
(SpMV, truncated Gram-Schmidt, SRHT, QR of the sketch, LSQR, f(C_m), the
final combination) runs in the library's CUDA kernels.

    op = Operator.stencil((g, g, g), coeffs)          # or Operator.csr(...)
    sv = Solver(op, b, m_max=200, k_max=4, s_max=400)
    sv.sketch(400, seed)          # before basis: fused sketch
    sv.basis(200, 4)              # Algorithm 2
    sv.compress("blendenpik")     # Algorithm 4 (or "sketch_solve", "none")
    y = sv.apply("sqrt", alpha=1.0, sigma=8080.08)
"""
import ctypes as C

import numpy as np

from . import _lib
from ._lib import (FabError, FabInfo, FabLsqrOpts, FabOperator, FabOpts, FUNCS, GET, MODES, check,
                   lib)

__all__ = ["Operator", "Solver", "FabError", "lib", "basis_batch", "solve"]


def _torch():
    import torch
    return torch


class Operator:
    """Device-side description of A (borrowed by the library)."""

    def __init__(self, st: FabOperator, keep=()):
        self.st = st
        self._keep = keep   # device tensors that must outlive the solver

    @property
    def n(self):
        return int(self.st.n)

    @staticmethod
    def stencil(dims, coeffs, rows=None):
        """Constant-coefficient stencil; rows = (row_begin, row_end) of this
        rank on several GPUs (dist.stencil_blocks), None = all rows."""
        st = FabOperator()
        st.kind = _lib.FAB_OP_STENCIL
        gx, gy, gz = (list(dims) + [1, 1])[:3]
        st.n = gx * gy * gz
        st.row_begin, st.row_end = (0, st.n) if rows is None else rows
        st.dims[:] = [gx, gy, gz]
        st.coeffs[:] = list(coeffs)
        st.value_scale = 1.0
        return Operator(st)

    @staticmethod
    def csr(indptr, indices, data=None, n=None, value_scale=1.0, device="cuda", rows=None):
        """CSR rows of A with GLOBAL column ids; rows = (row_begin, row_end)
        when these are one rank's block (dist.local_csr), n = global size."""
        torch = _torch()
        ip = torch.as_tensor(np.ascontiguousarray(indptr, dtype=np.int64)).to(device)
        ix = torch.as_tensor(np.ascontiguousarray(indices, dtype=np.int32)).to(device)
        dv = None
        if data is not None:
            dv = torch.as_tensor(np.ascontiguousarray(data, dtype=np.float64)).to(device)
        st = FabOperator()
        st.kind = _lib.FAB_OP_CSR
        nrows = len(indptr) - 1
        st.n = nrows if n is None else n
        st.row_begin, st.row_end = (0, nrows) if rows is None else rows
        assert st.row_end - st.row_begin == nrows
        st.nnz = int(indptr[-1])
        st.row_ptr = ip.data_ptr()
        st.col_idx = ix.data_ptr() if st.nnz else None
        st.values = dv.data_ptr() if dv is not None else None
        st.value_scale = value_scale
        return Operator(st, keep=(ip, ix, dv))

    @staticmethod
    def from_problem(p, csr=False, device="cuda"):
        """From a fab_problems.Problem (stencils stay matrix-free unless csr=True)."""
        if p.kind == "stencil" and not csr:
            return Operator.stencil(p.dims, p.coeffs)
        ip, ix, dv = p.csr()
        return Operator.csr(ip, ix, dv, device=device)


class Solver:
    def __init__(self, op: Operator, b, m_max, k_max=2, s_max=0, stream=None, device=None,
                 workspace=True, profile=False, comm=None, square=False, asynchronous=False):
        """b: this rank's rows (numpy host array or CUDA float64 tensor).
        comm: dist.Comm for a row-partitioned multi-GPU solve (every rank
        makes the same calls in the same order), None on one GPU.
        square: Krylov space of A^2 started from A b (FAB_FLAG_SQUARE), so
        apply("sign") = (A^2)^{-1/2} (A b) = sign(A) b.
        asynchronous: FAB_FLAG_ASYNC -- basis() and compress() only enqueue;
        their status is resolved (and returned) by apply() / get()."""
        torch = _torch()
        self.op = op
        self.torch = torch
        dev = torch.cuda.current_device() if device is None else device
        self.device = dev
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        o = FabOpts()
        o.stream = self.stream.cuda_stream
        o.device = dev
        o.m_max, o.k_max, o.s_max = m_max, k_max, s_max
        o.b_location = _lib.FAB_DEVICE
        o.flags = ((_lib.FAB_FLAG_PROFILE if profile else 0) | (_lib.FAB_FLAG_SQUARE if square else 0)
                   | (_lib.FAB_FLAG_ASYNC if asynchronous else 0))
        self.comm = comm
        o.comm = comm.handle.value if comm is not None else None
        if isinstance(b, np.ndarray):
            b = np.ascontiguousarray(b, dtype=np.float64)
            o.b_location = _lib.FAB_HOST
            bptr = b.ctypes.data
        else:
            assert b.dtype == torch.float64 and b.is_cuda and b.is_contiguous()
            bptr = b.data_ptr()
        self._ws = None
        if workspace:
            nbytes = C.c_size_t(0)
            check(lib.fab_workspace_size(C.byref(op.st), C.byref(o), C.byref(nbytes)), "fab_workspace_size")
            self._ws = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=f"cuda:{dev}")
            base = self._ws.data_ptr()
            o.workspace = (base + 255) // 256 * 256
            o.workspace_bytes = nbytes.value
        self.opts = o
        self.ctx = C.c_void_p()
        check(lib.fab_init(C.byref(self.ctx), C.byref(op.st), C.c_void_p(bptr), C.byref(o)), "fab_init")
        self.n = int(op.st.row_end - op.st.row_begin)
        self.status = {}

    # --- the five calls ---------------------------------------------------
    def basis(self, m, k):
        st = check(lib.fab_basis(self.ctx, m, k), "fab_basis")
        self.status["basis"] = st
        return st

    def basis_sgs(self, m):
        """Algorithm 1 (sketched Gram-Schmidt) with the Theta of sketch()."""
        st = check(lib.fab_basis_sgs(self.ctx, m), "fab_basis_sgs")
        self.status["basis"] = st
        return st

    def basis_whiten(self, m, k, cond_max=1000.0):
        """Algorithm 2 with whitening at cond > cond_max, then Algorithm 1."""
        st = check(lib.fab_basis_whiten(self.ctx, m, k, float(cond_max)), "fab_basis_whiten")
        self.status["basis"] = st
        return st

    def basis_arnoldi(self, m):
        """Full Arnoldi (CGS2), the paper's baseline; compress("none") = FOM."""
        st = check(lib.fab_basis_arnoldi(self.ctx, m), "fab_basis_arnoldi")
        self.status["basis"] = st
        return st

    def sketch(self, s, seed):
        st = check(lib.fab_sketch(self.ctx, s, C.c_uint64(seed)), "fab_sketch")
        self.status["sketch"] = st
        return st

    def compress(self, mode="blendenpik", iters=0, tol=0.0, maxit=0, precond_s=0, precond_seed=-1):
        """precond_s / precond_seed: Blendenpik's own preconditioner sketch
        Theta' (reading G-12); defaults reuse the Theta of sketch()."""
        o = FabLsqrOpts(iters, maxit, tol, precond_s, precond_seed)
        st = check(lib.fab_compress(self.ctx, MODES[mode], C.byref(o)), "fab_compress")
        self.status["compress"] = st
        return st

    def set_b(self, b):
        """Replace b (numpy host array or CUDA tensor); A and the sketch stay."""
        if isinstance(b, np.ndarray):
            check(lib.fab_set(self.ctx, _lib.FAB_SET_B_HOST, C.c_void_p(b.ctypes.data), b.nbytes), "fab_set(b)")
        else:
            check(lib.fab_set(self.ctx, _lib.FAB_SET_B_DEVICE, C.c_void_p(b.data_ptr()),
                              b.numel() * 8), "fab_set(b)")

    def set_poly(self, coef):
        a = np.ascontiguousarray(coef, dtype=np.float64)
        check(lib.fab_set(self.ctx, _lib.FAB_SET_POLY, C.c_void_p(a.ctypes.data), a.nbytes), "fab_set")

    def apply(self, f="exp", alpha=1.0, sigma=0.0, out=None, host=False):
        torch = self.torch
        if host:
            y = np.empty(self.n) if out is None else out
            ptr, loc = y.ctypes.data, _lib.FAB_HOST
        else:
            y = torch.empty(self.n, dtype=torch.float64, device=f"cuda:{self.device}") if out is None else out
            ptr, loc = y.data_ptr(), _lib.FAB_DEVICE
        st = check(lib.fab_apply(self.ctx, FUNCS[f], float(alpha), float(sigma), C.c_void_p(ptr), loc), "fab_apply")
        self.status["apply"] = st
        return y

    # --- results ------------------------------------------------------------
    def info(self):
        inf = FabInfo()
        check(lib.fab_get(self.ctx, GET["info"], C.byref(inf), C.sizeof(inf)), "fab_get")
        return inf.as_dict()

    def get(self, what):
        inf = self.info()
        me, n, s, N = inf["m_eff"], self.n, inf["s"], inf["N"]
        bd = inf["breakdown"]
        shapes = {
            "H": ((me, me + 1), np.float64), "V": ((me if bd else me + 1, n), np.float64),
            "SV": ((me if bd else me + 1, s), np.float64), "rows": ((s,), np.int64),
            "signs": (((N + 31) // 32,), np.uint32), "y": ((me,), np.float64),
            "C": ((me, me), np.float64), "fc": ((me,), np.float64), "R": ((me, me), np.float64),
            "beta": ((me + 1,), np.float64),
        }
        shape, dt = shapes[what]   # column-major matrices are allocated (cols, rows)
        a = np.empty(shape, dtype=dt)
        check(lib.fab_get(self.ctx, GET[what], C.c_void_p(a.ctypes.data), a.nbytes), f"fab_get({what})")
        if what in ("H", "V", "SV", "C", "R"):
            a = a.T.copy() if a.ndim == 2 else a     # column-major -> (rows, cols)
        return a

    def column(self, j):
        a = np.empty(self.n)
        check(lib.fab_get_column(self.ctx, j, C.c_void_p(a.ctypes.data)), "fab_get_column")
        return a

    def vrows(self, rows):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        inf = self.info()
        cols = inf["m_eff"] if inf["breakdown"] else inf["m_eff"] + 1
        a = np.empty((len(rows), cols))
        check(lib.fab_get_vrows(self.ctx, C.c_void_p(rows.ctypes.data), len(rows),
                                C.c_void_p(a.ctypes.data)), "fab_get_vrows")
        return a

    def close(self):
        if self.ctx:
            lib.fab_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def basis_batch(solvers, m, k):
    """Multi-RHS: Algorithm 2 for several Solvers of the same Operator at once
    (fab_basis_batch: one pass over the CSR entries per Krylov step for all
    of them); each Solver ends as after its own .basis(m, k)."""
    arr = (C.c_void_p * len(solvers))(*[sv.ctx.value for sv in solvers])
    st = check(lib.fab_basis_batch(arr, len(solvers), m, k), "fab_basis_batch")
    for sv in solvers:
        sv.status["basis"] = st
    return st


def solve(problem, mode="blendenpik", lsqr_iters=0, lsqr_tol=0.0, fused=True, csr=False):
    """One full f(A)b approximation of a fab_problems.Problem on cuda:0
    (convenience for tests / smoke)."""
    torch = _torch()
    op = Operator.from_problem(problem, csr=csr)
    b = torch.as_tensor(problem.b).cuda()
    sv = Solver(op, b, m_max=problem.m, k_max=problem.k, s_max=problem.s)
    if mode != "none" and fused:
        sv.sketch(problem.s, problem.sketch_seed)
    sv.basis(problem.m, problem.k)
    if mode != "none" and not fused:
        sv.sketch(problem.s, problem.sketch_seed)
    sv.compress(mode, iters=lsqr_iters, tol=lsqr_tol)
    y = sv.apply(problem.f, problem.alpha, problem.sigma)
    return y, sv

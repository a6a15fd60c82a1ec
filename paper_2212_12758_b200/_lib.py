"""ctypes binding of libfab.so (include/fab.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no
CPU fallback -- importing this module fails loudly if the library is missing.
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfab.so")
# profiling A/B only (profiles/build_variant.py): another build of the same library
if os.environ.get("FAB_LIB_VARIANT"):
    LIB_PATH = os.environ["FAB_LIB_VARIANT"]

# status codes (fab.h)
FAB_OK, FAB_BREAKDOWN, FAB_ILLCOND, FAB_NOTCONV = 0, 1, 2, 3
FAB_EINVAL, FAB_EORDER, FAB_ESINGULAR, FAB_EDOMAIN = -1, -2, -3, -4
FAB_ENOCONV, FAB_ENOMEM, FAB_ECUDA, FAB_ENCCL, FAB_ENODEV = -5, -6, -7, -8, -9
FAB_BLENDENPIK, FAB_SKETCH_SOLVE, FAB_NONE, FAB_LSQR, FAB_BLENDENPIK_GRAM = 0, 1, 2, 3, 4
FAB_EXP, FAB_SQRT, FAB_INVSQRT, FAB_POLY, FAB_SIGN = 0, 1, 2, 3, 4
FAB_OP_CSR, FAB_OP_STENCIL = 0, 1
FAB_DEVICE, FAB_HOST = 0, 1
GET = dict(info=0, H=1, V=2, SV=3, rows=4, signs=5, y=6, C=7, fc=8, R=9, beta=10)
FAB_SET_POLY, FAB_SET_B_HOST, FAB_SET_B_DEVICE = 100, 101, 102
FAB_FLAG_PROFILE, FAB_FLAG_SQUARE, FAB_FLAG_ASYNC = 1, 2, 4

MODES = {"blendenpik": FAB_BLENDENPIK, "sketch_solve": FAB_SKETCH_SOLVE, "none": FAB_NONE, "lsqr": FAB_LSQR,
         "blendenpik_gram": FAB_BLENDENPIK_GRAM}
FUNCS = {"exp": FAB_EXP, "sqrt": FAB_SQRT, "invsqrt": FAB_INVSQRT, "poly": FAB_POLY, "sign": FAB_SIGN}

# every function declared in include/fab.h
EXPORTS = ("fab_version", "fab_strerror", "fab_workspace_size", "fab_init", "fab_basis", "fab_basis_batch",
           "fab_basis_sgs", "fab_basis_arnoldi", "fab_basis_whiten",
           "fab_sketch", "fab_compress", "fab_apply", "fab_get", "fab_get_column", "fab_get_vrows",
           "fab_set", "fab_last_error", "fab_destroy", "fab_comm_unique_id", "fab_comm_init",
           "fab_comm_init_loopback", "fab_comm_p2p", "fab_comm_destroy")


class FabOperator(C.Structure):
    _fields_ = [("kind", C.c_int), ("row_ptr_64", C.c_int), ("n", C.c_int64),
                ("row_begin", C.c_int64), ("row_end", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p),
                ("value_scale", C.c_double), ("dims", C.c_int64 * 3), ("coeffs", C.c_double * 7)]


class FabOpts(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("device", C.c_int), ("m_max", C.c_int),
                ("k_max", C.c_int), ("s_max", C.c_int), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("b_location", C.c_int), ("flags", C.c_uint),
                ("comm", C.c_void_p)]


class FabLsqrOpts(C.Structure):
    _fields_ = [("iters", C.c_int), ("maxit", C.c_int), ("tol", C.c_double), ("precond_s", C.c_int),
                ("precond_pad", C.c_int), ("precond_seed", C.c_int64)]

    def __init__(self, iters=0, maxit=0, tol=0.0, precond_s=0, precond_seed=-1):
        super().__init__(iters, maxit, tol, precond_s, 0, precond_seed)


class FabInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("N", C.c_int64), ("m", C.c_int), ("k", C.c_int), ("s", C.c_int),
                ("m_eff", C.c_int), ("breakdown", C.c_int), ("sketch_fused", C.c_int),
                ("mode", C.c_int), ("lsqr_iters", C.c_int), ("lsqr_converged", C.c_int),
                ("dense_iters", C.c_int), ("basis_alg", C.c_int), ("gamma_b", C.c_double),
                ("h_last", C.c_double), ("norm_inf", C.c_double), ("cond_R", C.c_double),
                ("lsqr_rnorm", C.c_double), ("lsqr_arnorm", C.c_double), ("lsqr_anorm", C.c_double),
                ("ms_basis", C.c_double), ("ms_sketch", C.c_double), ("ms_compress", C.c_double),
                ("ms_apply", C.c_double), ("launches_basis", C.c_int64),
                ("launches_sketch", C.c_int64), ("launches_compress", C.c_int64),
                ("launches_apply", C.c_int64), ("ms_lsqr_pass", C.c_double),
                ("lsqr_passes", C.c_int64), ("ms_sketch_batched", C.c_double),
                ("whitened_at", C.c_int), ("pad1", C.c_int), ("whiten_cond", C.c_double),
                ("gram_used", C.c_int), ("pad2", C.c_int), ("precond_s", C.c_int),
                ("precond_fresh", C.c_int), ("ms_precond_sketch", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k not in ("pad1", "pad2")}


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with `python -m paper_2212_12758_b200._build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I, D = C.c_void_p, C.c_int, C.c_double
    sig = {
        "fab_version": (I, []),
        "fab_strerror": (C.c_char_p, [I]),
        "fab_last_error": (C.c_char_p, []),
        "fab_workspace_size": (I, [C.POINTER(FabOperator), C.POINTER(FabOpts), C.POINTER(C.c_size_t)]),
        "fab_init": (I, [C.POINTER(P), C.POINTER(FabOperator), P, C.POINTER(FabOpts)]),
        "fab_basis": (I, [P, I, I]),
        "fab_basis_batch": (I, [C.POINTER(P), I, I, I]),
        "fab_basis_sgs": (I, [P, I]),
        "fab_basis_arnoldi": (I, [P, I]),
        "fab_basis_whiten": (I, [P, I, I, D]),
        "fab_sketch": (I, [P, I, C.c_uint64]),
        "fab_compress": (I, [P, I, C.POINTER(FabLsqrOpts)]),
        "fab_apply": (I, [P, I, D, D, P, I]),
        "fab_get": (I, [P, I, P, C.c_size_t]),
        "fab_set": (I, [P, I, P, C.c_size_t]),
        "fab_get_column": (I, [P, I, P]),
        "fab_get_vrows": (I, [P, P, I, P]),
        "fab_destroy": (I, [P]),
        "fab_comm_unique_id": (I, [P]),
        "fab_comm_init": (I, [C.POINTER(P), P, I, I, I]),
        "fab_comm_init_loopback": (I, [P, I, I]),
        "fab_comm_p2p": (I, [P]),
        "fab_comm_destroy": (I, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


class FabError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = lib.fab_strerror(status).decode()
        super().__init__(f"{where}: status {status}: {msg}")


def check(status, where, allow_warn=True):
    if status < 0 or (status > 0 and not allow_warn):
        raise FabError(status, where)
    return status

"""Row-partitioned multi-GPU support: host logic
only -- partition plans, local operators, and the NCCL communicator
bootstrap.  Every collective of the path itself is issued by libfab.so
(comm.cu); this module never touches the data.

One process per GPU.  Rank p owns rows [rows[p], rows[p+1]) of A, b, V and
f_m.  Boundaries are multiples of 32 rows (256-B aligned bulk copies; the
stencil kernel's double2 row pairs), every block holds at least the halo
(one grid plane for a 3D stencil), and the blocks tile [0, n) in rank order.
"""
import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib

ALIGN = 32


def stencil_halo(dims):
    """Widest stencil offset (rows): one plane in 3D, one line in 2D."""
    gx, gy, gz = (list(dims) + [1, 1])[:3]
    return gx * gy if gz > 1 else (gx if gy > 1 else 1)


def _aligned_cuts(targets, n, align):
    cuts = [0]
    for t in targets:
        c = int(round(t / align)) * align
        cuts.append(min(max(c, cuts[-1]), n))
    cuts.append(n)
    return np.asarray(cuts, dtype=np.int64)


def row_blocks(n, nranks, align=ALIGN, min_rows=1):
    """Equal contiguous row blocks with 32-aligned starts (c5: uniform rows)."""
    cuts = _aligned_cuts([p * n / nranks for p in range(1, nranks)], n, align)
    _check(cuts, n, min_rows)
    return cuts


def stencil_blocks(dims, nranks):
    """z-slabs (3D) / y-bands (2D) of whole grid planes / lines, as equal as
    possible (c3: 256 planes over P ranks -> 256/P planes each)."""
    gx, gy, gz = (list(dims) + [1, 1])[:3]
    unit = gx * gy if gz > 1 else gx           # rows per plane (3D) or line (2D)
    count = gz if gz > 1 else gy
    if count < nranks:
        raise ValueError(f"{count} planes cannot be split over {nranks} ranks")
    base, extra = divmod(count, nranks)
    sizes = [base + (1 if p < extra else 0) for p in range(nranks)]
    cuts = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64) * unit
    if any(c % ALIGN for c in cuts[:-1]):
        # planes not 32-aligned: fall back to aligned row blocks
        cuts = row_blocks(gx * gy * gz, nranks, ALIGN, stencil_halo(dims))
    _check(cuts, gx * gy * gz, stencil_halo(dims))
    return cuts


def csr_blocks(indptr, nranks, align=ALIGN):
    """nnz-balanced contiguous row blocks (c4: power-law hubs sit at low row
    ids, so equal row counts would be badly imbalanced)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    n = len(indptr) - 1
    nnz = int(indptr[-1])
    targets = []
    for p in range(1, nranks):
        r = int(np.searchsorted(indptr, p * nnz / nranks))
        targets.append(min(r, n))
    cuts = _aligned_cuts(targets, n, align)
    _check(cuts, n, 1)
    return cuts


def _check(cuts, n, min_rows):
    cuts = np.asarray(cuts)
    if cuts[0] != 0 or cuts[-1] != n:
        raise ValueError("blocks must tile [0, n)")
    if any(c % ALIGN for c in cuts[:-1]):
        raise ValueError("block starts must be multiples of 32 rows")
    if np.any(np.diff(cuts) < min_rows):
        raise ValueError(f"every block needs >= {min_rows} rows (halo); use fewer ranks")


def local_csr(indptr, indices, data, r0, r1):
    """Rows [r0, r1) of a CSR matrix with GLOBAL column ids (rebased row_ptr)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    a, b = int(indptr[r0]), int(indptr[r1])
    ip = indptr[r0:r1 + 1] - a
    ix = np.asarray(indices[a:b], dtype=np.int32)
    dv = None if data is None else np.asarray(data[a:b], dtype=np.float64)
    return ip, ix, dv


def local_operator(problem, r0, r1, csr=False, device="cuda"):
    """The operator of rank with rows [r0, r1) (stencils stay matrix-free)."""
    from . import Operator
    if problem.kind == "stencil" and not csr:
        return Operator.stencil(problem.dims, problem.coeffs, rows=(r0, r1))
    ip, ix, dv = problem.csr()
    lip, lix, ldv = local_csr(ip, ix, dv, r0, r1)
    return Operator.csr(lip, lix, ldv, n=problem.n, rows=(r0, r1), device=device)


class Comm:
    """NCCL communicator of libfab.so for the ranks of a torch.distributed
    group: rank 0 draws the NCCL unique id, torch broadcasts it."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else device
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            check(lib.fab_comm_unique_id(C.cast(uid, C.c_void_p)), "fab_comm_unique_id")
        obj = [uid.raw if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = C.create_string_buffer(obj[0], 128)
        self.handle = C.c_void_p()
        check(lib.fab_comm_init(C.byref(self.handle), C.cast(uid, C.c_void_p), self.rank, self.size,
                                self.device), "fab_comm_init")

    @property
    def p2p(self):
        """True if C2 runs through the NVLink mailboxes (fab_comm_p2p)."""
        return bool(lib.fab_comm_p2p(self.handle))

    def close(self):
        if self.handle:
            lib.fab_comm_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackComm:
    """One rank of a loopback group (fab_comm_init_loopback): same interface
    as Comm (.rank, .size, .handle); owned by its LoopbackGroup."""

    def __init__(self, handle, rank, size, device):
        self.handle = C.c_void_p(handle)
        self.rank, self.size, self.device = rank, size, device

    def close(self):
        if self.handle:
            lib.fab_comm_destroy(self.handle)
            self.handle = C.c_void_p()


class LoopbackGroup:
    """P ranks of one row-partitioned solve on ONE GPU (SURVEY §4 tier T3'):
    the path's halo / all-gather / allreduce data movement without NCCL.
    Drive rank r from its own host thread and its own CUDA stream (`run`)."""

    def __init__(self, nranks, device=0):
        arr = (C.c_void_p * nranks)()
        check(lib.fab_comm_init_loopback(C.cast(arr, C.c_void_p), nranks, device), "fab_comm_init_loopback")
        self.comms = [LoopbackComm(arr[r], r, nranks, device) for r in range(nranks)]

    def run(self, fn):
        """fn(rank, comm, stream) on P threads at once; returns the P results
        (re-raises the first exception)."""
        import threading

        import torch
        out = [None] * len(self.comms)
        errs = [None] * len(self.comms)
        dev = self.comms[0].device

        def body(r):
            try:
                torch.cuda.set_device(dev)
                st = torch.cuda.Stream(device=dev)
                with torch.cuda.stream(st):
                    out[r] = fn(r, self.comms[r], st)
                st.synchronize()
            except BaseException as e:   # noqa: BLE001
                errs[r] = e
        ts = [threading.Thread(target=body, args=(r,)) for r in range(len(self.comms))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in errs:
            if e is not None:
                raise e
        return out

    def close(self):
        for cm in self.comms:
            cm.close()


__all__ = ["Comm", "LoopbackGroup", "LoopbackComm", "row_blocks", "stencil_blocks", "csr_blocks", "local_csr", "local_operator",
           "stencil_halo", "ALIGN"]
_ = _lib

"""CPU-side checks of the C ABI: libfab.so loads, exports every function that
include/fab.h declares, and its host-side validation / status logic works
without a GPU (no compute calls)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "fab.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(fab_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2212_12758_b200 import _lib
    names = header_functions()
    assert len(names) >= 12
    lib = C.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTS)


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors of fab_operator / fab_opts / fab_lsqr_opts /
    fab_info have the C compiler's size and every field's offset (gcc on
    include/fab.h), so the binding marshals exactly what the ABI declares."""
    import subprocess
    from paper_2212_12758_b200 import _lib
    structs = {"fab_operator": _lib.FabOperator, "fab_opts": _lib.FabOpts, "fab_lsqr_opts": _lib.FabLsqrOpts,
               "fab_info": _lib.FabInfo}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "fab.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["return 0; }"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(ln.split()[:2]): int(ln.split()[2]) for ln in out if ln.strip()}
    for cname, py in structs.items():
        assert got[(cname, "sizeof")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


def test_version_and_strerror():
    from paper_2212_12758_b200 import _lib
    assert _lib.lib.fab_version() == 2
    for code in (0, 1, 2, 3, -1, -2, -3, -4, -5, -6, -7, -8, -9):
        assert len(_lib.lib.fab_strerror(code)) > 0
    assert _lib.lib.fab_strerror(12345) == b"unknown status"


def _stencil_op(g=8):
    from paper_2212_12758_b200 import _lib
    st = _lib.FabOperator()
    st.kind = _lib.FAB_OP_STENCIL
    st.n = g * g
    st.row_begin, st.row_end = 0, g * g
    st.dims[:] = [g, g, 1]
    st.coeffs[:] = [4, -1, -1, -1, -1, 0, 0]
    return st


def _opts(m=4, k=2, s=8):
    from paper_2212_12758_b200 import _lib
    o = _lib.FabOpts()
    o.device = -1
    o.m_max, o.k_max, o.s_max = m, k, s
    return o


def test_validation_without_device():
    from paper_2212_12758_b200 import _lib
    lib = _lib.lib
    nb = C.c_size_t(0)
    st = _stencil_op()
    # invalid capacities are rejected before any device query
    for bad in [dict(m=0), dict(m=64), dict(k=0), dict(k=9), dict(s=-1), dict(s=10000)]:
        kw = dict(m=4, k=2, s=8)
        kw.update(bad)
        assert lib.fab_workspace_size(C.byref(st), C.byref(_opts(**kw)), C.byref(nb)) == _lib.FAB_EINVAL
    bad = _stencil_op()
    bad.dims[:] = [3, 3, 1]          # dims inconsistent with n
    assert lib.fab_workspace_size(C.byref(bad), C.byref(_opts()), C.byref(nb)) == _lib.FAB_EINVAL
    bad = _stencil_op()
    bad.kind = 7
    assert lib.fab_workspace_size(C.byref(bad), C.byref(_opts()), C.byref(nb)) == _lib.FAB_EINVAL
    csr = _lib.FabOperator()
    csr.kind = _lib.FAB_OP_CSR
    csr.n = 10
    csr.row_end = 10
    assert lib.fab_workspace_size(C.byref(csr), C.byref(_opts()), C.byref(nb)) == _lib.FAB_EINVAL
    # null context / pointers
    assert lib.fab_basis(None, 4, 2) == _lib.FAB_EINVAL
    assert lib.fab_destroy(None) == _lib.FAB_EINVAL
    # multi-RHS batch: null array, bad counts, null members
    assert lib.fab_basis_batch(None, 1, 4, 2) == _lib.FAB_EINVAL
    arr = (C.c_void_p * 5)()
    assert lib.fab_basis_batch(arr, 0, 4, 2) == _lib.FAB_EINVAL
    assert lib.fab_basis_batch(arr, 5, 4, 2) == _lib.FAB_EINVAL
    assert lib.fab_basis_batch(arr, 2, 4, 2) == _lib.FAB_EINVAL          # null contexts
    # sign needs a squared context; apply on a null context is rejected first
    assert lib.fab_apply(None, _lib.FAB_SIGN, 1.0, 0.0, None, 0) == _lib.FAB_EINVAL


def test_init_reports_no_device_on_cpu_box():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2212_12758_b200 import _lib
    import numpy as np
    b = np.ones(64)
    ctx = C.c_void_p()
    rc = _lib.lib.fab_init(C.byref(ctx), C.byref(_stencil_op()), C.c_void_p(b.ctypes.data),
                           C.byref(_opts()))
    assert rc in (_lib.FAB_ENODEV, _lib.FAB_ECUDA)
    assert not ctx.value


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2212_12758_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f

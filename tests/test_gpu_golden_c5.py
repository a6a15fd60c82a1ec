"""Element-wise oracle parity at BASELINE.json c5 at full size: n = 2^25
random nonsymmetric sparse (570 M entries; on the GPU the column-blocked
CSR K1, 6 passes per product), f = (-A)^{-1/2}, m = 300, k = 2, s = 600 --
the largest configuration, V_{m+1} = 80.8 GB in HBM.

Expected values: tests/golden/c5_full.npz, written by the oracle-only script
tests/golden/make_c5_golden.py (its V_{m+1} in a memory map on disk).  The
basis is well conditioned (cond(Theta V_m) ~ 5.5), so H and the
sketch-and-solve y are determined: held to 1e-12 / 1e-10; f_m (converged,
~5^-m) per mode on every 8192nd row, on the sums of all 4096 blocks of 8192
rows and its norm: 1e-10.  Tolerance-mode Blendenpik: the oracle's
iteration count (+-1) and f_m at 1e-10; its y is an unconverged iterate
(reading R-3) and is compared loosely (1e-5).
"""
import json
import os

import numpy as np
import pytest

import fab_problems as fp

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c5_full.npz")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def run():
    import hashlib

    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(GOLDEN):
        pytest.fail(f"{GOLDEN} missing: run tests/golden/make_c5_golden.py (oracle only)")
    torch.cuda.set_device(0)
    torch.cuda.empty_cache()
    import paper_2212_12758_b200 as fab
    g = dict(np.load(GOLDEN))
    meta = json.loads(bytes(g["meta_json"]).decode())
    p = fp.make("c5")
    assert hashlib.sha256(np.ascontiguousarray(p.b).tobytes()).hexdigest() == meta["b_sha256"]
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
    y = torch.empty(p.n, dtype=torch.float64, device="cuda")
    res = {}
    for key, kw in {"none": dict(mode="none"), "sketch_solve": dict(mode="sketch_solve"),
                    "blendenpik": dict(mode="blendenpik", tol=1e-6)}.items():
        if kw["mode"] != "none":
            sv.sketch(p.s, p.sketch_seed)
        sv.basis(p.m, p.k)
        sv.compress(kw["mode"], tol=kw.get("tol", 0.0))
        sv.apply(p.f, p.alpha, p.sigma, out=y)
        fm = y.cpu().numpy()
        nb = p.n // meta["block"]
        res[key] = dict(samples=fm[::meta["stride"]].copy(),
                        blocks=fm[: nb * meta["block"]].reshape(nb, meta["block"]).sum(axis=1),
                        norm=np.linalg.norm(fm), H=sv.get("H"), y=sv.get("y"), c=sv.get("fc"),
                        info=sv.info(), rows=sv.get("rows") if key != "none" else None)
        del fm
    yield p, g, meta, res
    sv.close()
    del y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("key", ["none", "sketch_solve", "blendenpik"])
def test_c5_fm_per_mode(run, key):
    p, g, meta, res = run
    r = res[key]
    assert rel(r["samples"], g[f"{key}_fm_samples"]) <= 1e-10
    assert rel(r["blocks"], g[f"{key}_fm_blocks"]) <= 1e-10
    assert abs(r["norm"] - float(g[f"{key}_fm_norm"])) <= 1e-10 * float(g[f"{key}_fm_norm"])


def test_c5_basis_compression(run):
    p, g, meta, res = run
    assert rel(res["none"]["H"], g["H"]) <= 1e-12
    assert np.array_equal(res["sketch_solve"]["rows"], g["rows"])
    assert rel(res["sketch_solve"]["y"], g["sketch_solve_y"]) <= 1e-10
    assert rel(res["sketch_solve"]["c"], g["sketch_solve_c"]) <= 1e-10
    assert rel(res["none"]["c"], g["none_c"]) <= 1e-10
    b = res["blendenpik"]
    L = int(meta["blendenpik_lsqr"]["iters"])
    assert b["info"]["lsqr_converged"] == 1 and abs(b["info"]["lsqr_iters"] - L) <= 1
    assert rel(b["y"], g["blendenpik_y"]) <= 1e-5

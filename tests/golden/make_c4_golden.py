#!/usr/bin/env python
"""Full-size BASELINE.json c4 oracle outputs for tests/test_gpu_golden_c4.py:
the random-graph workload of the north star at its own size (the CSR path,
nnz-balanced row blocks, uniform-value entries) compared element-wise.

Calls ONLY oracle/ and the seeded generator fab_problems (plus scipy's
expm_multiply for the exact f(A)b, "exact" reference).

    python tests/golden/make_c4_golden.py [--out tests/golden/c4_full.npz]

Workload: c4 = Chung-Lu power-law graph, n = 2^22, mean degree 12, A/lambda_hat
(reading G-25), b = +-1/sqrt(n), f = exp, m = 150, k = 2, s = 300.  The
Krylov space saturates near m = 30 (cond(Theta V_m) ~ 1e15 at m = 150:
SURVEY §8c-4), so y and the late basis are NOT determined by the data
(reading G-24) -- only f_m is, and it has converged: the file keeps, per mode
(Algorithm 5, sketch-and-solve, Blendenpik at tol 1e-6), f_m on every 1024th
row, the sums of the 4096 blocks of 1024 rows and ||f_m||, the same for the
exact exp(A) b, and underline-H_m (whose first columns are determined).
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import scipy.sparse.linalg as spla  # noqa: E402

import fab_problems as fp  # noqa: E402
from oracle import fab as ofab  # noqa: E402
from oracle import krylov, matfun  # noqa: E402
from oracle.srht import SRHT  # noqa: E402

STRIDE = 1024
BLOCK = 1024


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def summary(v):
    nb = v.shape[0] // BLOCK
    return dict(samples=v[::STRIDE].copy(), blocks=v[: nb * BLOCK].reshape(nb, BLOCK).sum(axis=1),
                norm=np.array(np.linalg.norm(v)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c4_full.npz"))
    ap.add_argument("--n", type=int, default=1 << 22)
    args = ap.parse_args()
    t_all = time.perf_counter()
    p = fp.make("c4", n=args.n)
    A = p.scipy()
    log(f"[golden c4] n={p.n} nnz={A.nnz} m={p.m} k={p.k} s={p.s}")
    t0 = time.perf_counter()
    exact = spla.expm_multiply(p.alpha * A, p.b)                                # exp(A) b
    log(f"[golden c4] expm_multiply {time.perf_counter() - t0:.1f} s")
    t0 = time.perf_counter()
    dec = krylov.truncated_arnoldi(A, p.b, p.m, p.k, variant="cgs")             # Algorithm 2
    log(f"[golden c4] basis {time.perf_counter() - t0:.1f} s, m_eff={dec['m_eff']}")
    V, m = dec["V"], dec["m_eff"]
    t0 = time.perf_counter()
    th = SRHT(p.n, p.s, p.sketch_seed)
    SV = th.apply(V)
    log(f"[golden c4] SRHT {time.perf_counter() - t0:.1f} s")
    out = dict(H=dec["H"], rows=th.rows)
    for kk, vv in summary(exact).items():
        out[f"exact_{kk}"] = vv
    meta = dict(config="c4", n=p.n, m=p.m, k=p.k, s=p.s, seed=p.sketch_seed, f=p.f, alpha=p.alpha,
                breakdown=bool(dec["breakdown"]), m_eff=m, stride=STRIDE, block=BLOCK,
                b_sha256=hashlib.sha256(np.ascontiguousarray(p.b).tobytes()).hexdigest())
    modes = {"none": dict(mode="none"), "sketch_solve": dict(mode="sketch_solve"),
             "blendenpik": dict(mode="blendenpik", lsqr_tol=1e-6)}
    for key, kw in modes.items():
        t0 = time.perf_counter()
        y, C, R, info = ofab.compress(dec, SV, kw["mode"], lsqr_tol=kw.get("lsqr_tol", 1e-6))
        c = matfun.f_e1(p.f, C, p.alpha, p.sigma)
        fm = dec["gamma"] * (V[:, :m] @ c)
        for kk, vv in summary(fm).items():
            out[f"{key}_fm_{kk}"] = vv
        meta[f"{key}_lsqr"] = {kk: (float(vv) if not isinstance(vv, bool) else vv) for kk, vv in (info or {}).items()}
        meta[f"{key}_err_vs_exact"] = float(np.linalg.norm(fm - exact) / np.linalg.norm(exact))
        log(f"[golden c4] {key}: {time.perf_counter() - t0:.1f} s, rel. err vs exact "
            f"{meta[key + '_err_vs_exact']:.2e}, lsqr={meta[key + '_lsqr']}")
        del fm
    meta["seconds"] = time.perf_counter() - t_all
    out["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(args.out, **out)
    log(f"[golden c4] wrote {args.out} ({os.path.getsize(args.out) / 1e6:.2f} MB) in {meta['seconds']:.0f} s")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Full-size BASELINE.json c3 oracle outputs for the GPU parity test
tests/test_gpu_golden_c3.py (VERDICT r01 "next" #1: an element-wise oracle
comparison at the headline configuration).

Calls ONLY oracle/ (the fp64 CPU implementation written from the paper) and
the seeded input generator fab_problems; nothing from the CUDA path.

    python tests/golden/make_c3_golden.py [--out tests/golden/c3_full.npz]

Workload: c3 = 3D upwind convection-diffusion 256^3 (n = 2^24), seeded
Gaussian b, m = 200, k = 4, s = 400, f = sqrt with sigma = 1e-2 ||A||_inf.
Steps, each the oracle's own (no shortcuts):
  * Algorithm 2, variant "cgs" (reading G-2: the GPU's
    one-pass CGS in the window) -> V_{m+1}, underline-H_m, gamma = ||b||
  * Theta V_{m+1} with the SRHT of l.70 (oracle/srht.py, readings G-6..G-10)
  * the compression of Eq. (6)/(7) in four modes (l.174-184, l.199-209,
    l.211-228, l.249-251):
        none          Algorithm 5 (y = 0)
        sketch_solve  Remark 2 (y = R^{-1} Q^T Theta v_{m+1})
        blendenpik40  Blendenpik-LSQR with exactly L = 40 iterations (G-14)
        blendenpik    Blendenpik-LSQR at the MATLAB tolerance 1e-6 (l.359)
        blendenpik120 Blendenpik-LSQR with L = 120 iterations: converged to
                      the least-squares solution (contraction ~0.7 per
                      iteration at s = 2m), so y is determined by the data
        blendenpik40_inv  the L = 40 run with R^{-1} applied as an explicit
                      inverse instead of by substitution: the same method in
                      other rounding -- its distance to blendenpik40 is the
                      oracle's own noise floor for an unconverged iterate
                      (reading R-3)
  * c = sqrt(C_m + sigma I) e_1 (scipy sqrtm, l.356) and f_m = gamma V_m c
    (Algorithm 4 line 3, l.207).

f_m has 2^24 entries (128 MB), too large to commit; the file keeps, per mode,
every 4096th row (4096 values), the sums over the 4096 consecutive blocks of
4096 rows (every entry of f_m enters one of them), and ||f_m||.  The full
H, Theta V, R, y and c are kept.  Needs ~32 GB RAM and ~45 min on 8 cores.
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

import fab_problems as fp  # noqa: E402
from oracle import fab as ofab  # noqa: E402
from oracle import krylov, matfun  # noqa: E402
from oracle.srht import SRHT  # noqa: E402

STRIDE = 4096      # sampled rows of f_m: 0, 4096, 8192, ...
BLOCK = 4096       # block sums of f_m


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def fm_summary(fm):
    n = fm.shape[0]
    nb = n // BLOCK
    return dict(samples=fm[::STRIDE].copy(), blocks=fm[: nb * BLOCK].reshape(nb, BLOCK).sum(axis=1),
                norm=np.array(np.linalg.norm(fm)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c3_full.npz"))
    ap.add_argument("--g", type=int, default=256)
    args = ap.parse_args()
    t_all = time.perf_counter()
    p = fp.make("c3", g=args.g)
    A = p.scipy()
    log(f"[golden] c3 n={p.n} m={p.m} k={p.k} s={p.s} sigma={p.sigma}")
    t0 = time.perf_counter()
    dec = krylov.truncated_arnoldi(A, p.b, p.m, p.k, variant="cgs")          # Algorithm 2
    log(f"[golden] basis {time.perf_counter() - t0:.1f} s, m_eff={dec['m_eff']}")
    assert not dec["breakdown"]
    V, H, m = dec["V"], dec["H"], dec["m_eff"]
    t0 = time.perf_counter()
    th = SRHT(p.n, p.s, p.sketch_seed)
    SV = th.apply(V)                                                          # Theta V_{m+1}
    log(f"[golden] SRHT {time.perf_counter() - t0:.1f} s")
    out = dict(H=H, SV=SV, rows=th.rows, gamma=np.array(dec["gamma"]))
    # sampled rows of the normalized basis (both grid corners included)
    vr = np.unique(np.concatenate([[0, p.n - 1], np.random.default_rng(7).integers(0, p.n, 62)]))
    out["vrows_idx"] = vr
    out["vrows"] = V[vr, :].copy()
    meta = dict(config="c3", n=p.n, m=p.m, k=p.k, s=p.s, seed=p.sketch_seed, f=p.f, alpha=p.alpha,
                sigma=p.sigma, variant="cgs", stride=STRIDE, block=BLOCK,
                b_sha256=hashlib.sha256(np.ascontiguousarray(p.b).tobytes()).hexdigest(),
                signs_sha256=hashlib.sha256((th.signs < 0).astype(np.uint8).tobytes()).hexdigest())
    modes = {"none": dict(mode="none"), "sketch_solve": dict(mode="sketch_solve"),
             "blendenpik40": dict(mode="blendenpik", lsqr_iters=40),
             "blendenpik": dict(mode="blendenpik", lsqr_tol=1e-6),
             "blendenpik120": dict(mode="blendenpik", lsqr_iters=120),
             "blendenpik40_inv": dict(mode="blendenpik", lsqr_iters=40, rinv="inverse")}
    for key, kw in modes.items():
        t0 = time.perf_counter()
        y, C, R, info = ofab.compress(dec, SV, kw["mode"], lsqr_tol=kw.get("lsqr_tol", 1e-6),
                                      lsqr_iters=kw.get("lsqr_iters"), rinv=kw.get("rinv", "solve"))  # Eq. (6)/(7)
        c = matfun.f_e1(p.f, C, p.alpha, p.sigma)                              # f(C_m) e_1
        fm = dec["gamma"] * (V[:, :m] @ c)                                     # l.207
        s = fm_summary(fm)
        out[f"{key}_y"] = y
        out[f"{key}_c"] = c
        out[f"{key}_C_last"] = C[:, m - 1].copy()
        for kk, vv in s.items():
            out[f"{key}_fm_{kk}"] = vv
        if R is not None and "R" not in out:
            out["R"] = R
        meta[f"{key}_lsqr"] = {kk: (float(vv) if not isinstance(vv, bool) else vv)
                               for kk, vv in (info or {}).items()}
        log(f"[golden] {key}: {time.perf_counter() - t0:.1f} s, lsqr={meta[key + '_lsqr']}, "
            f"||f_m||={float(s['norm']):.6e}")
        del fm
    meta["seconds"] = time.perf_counter() - t_all
    out["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(args.out, **out)
    log(f"[golden] wrote {args.out} ({os.path.getsize(args.out) / 1e6:.2f} MB) in {meta['seconds']:.0f} s")


if __name__ == "__main__":
    main()

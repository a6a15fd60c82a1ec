"""Every BASELINE.json config at full size on one B200 (SURVEY.md §8(d-1):
"Every config is reported").  Side measurement next to bench.py (whose
headline line is c3); run on a GPU box:

    python profiles/bench_configs.py [c1 c2 c4 c5 c3] > gpurun_out/configs.jsonl

Per config, through the C ABI with A and b resident in HBM:
  * init_ms          fab_init (copies / validation / ||A||_inf), once
  * iters_per_s      m / T(fab_basis) with the sketch fused (fab_sketch first)
  * basis_gbs        algorithmic bytes per Krylov step (DESIGN.md §7:
                     8n(2k+3) + B_A, B_A = 8(n+1) + 12 nnz for CSR) / step time
  * solves_per_s     per mode: Blendenpik-LSQR at tol 1e-6, sketch-and-solve,
                     none (Algorithm 5); median of `reps` solves
  * lsqr_pass_gbs    8n(m+2) bytes / average fused LSQR pass time
  * mode_agreement   ||f_mode - f_blendenpik|| / ||f_blendenpik||
CUDA-event times come from the library (FAB_FLAG_PROFILE, events on its
stream).  The inputs are the fab_problems recipes (seeded, synthetic).
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def run(name, reps=3):
    t0 = time.perf_counter()
    p = fp.make(name)
    t_gen = time.perf_counter() - t0
    log(f"[{name}] generated n={p.n} in {t_gen:.1f} s")
    op = fab.Operator.from_problem(p)
    b = torch.as_tensor(p.b).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sv = fab.Solver(op, b, m_max=p.m, k_max=p.k, s_max=p.s, profile=True)
    torch.cuda.synchronize()
    init_ms = (time.perf_counter() - t0) * 1e3
    y = torch.empty(p.n, dtype=torch.float64, device="cuda")
    n, m, k, s = p.n, p.m, p.k, p.s
    if p.kind == "csr":
        nnz = int(p.meta["nnz"])
        dv = p.csr()[2]
        uniform = bool(len(dv) and np.all(dv == dv[0]))     # fab_init drops the value array then
        b_a = 8.0 * (n + 1) + (4.0 if uniform else 12.0) * nnz
    else:
        nnz = None
        b_a = 0.0
    b_it = 8.0 * n * (2 * k + 3) + b_a

    def solve(mode):
        if mode != "none":
            sv.sketch(s, p.sketch_seed)
        sv.basis(m, k)
        sv.compress(mode, tol=1e-6)
        sv.apply(p.f, p.alpha, p.sigma, out=y)
        return sv.info()

    out = {"config": name, "n": n, "m": m, "k": k, "s": s, "f": p.f, "alpha": p.alpha,
           "sigma": p.sigma, "kind": p.kind, "nnz": nnz, "gen_s": t_gen, "init_ms": init_ms,
           "meta": {kk: vv for kk, vv in p.meta.items() if isinstance(vv, (int, float, str))}}
    res = {}
    for mode in ("blendenpik", "sketch_solve", "none"):
        solve(mode)      # warm-up (graph capture, first touch)
        infs, tot = [], []
        for _ in range(reps):
            inf = solve(mode)
            infs.append(inf)
            tot.append(inf["ms_sketch"] + inf["ms_basis"] + inf["ms_compress"] + inf["ms_apply"])
        res[mode] = (y.cpu().numpy(), infs)
        med = statistics.median(tot)
        ent = {"solves_per_s": 1e3 / med, "ms_per_solve": med,
               "ms_basis": statistics.median(i["ms_basis"] for i in infs),
               "ms_compress": statistics.median(i["ms_compress"] for i in infs),
               "ms_apply": statistics.median(i["ms_apply"] for i in infs),
               "m_eff": infs[-1]["m_eff"], "breakdown": infs[-1]["breakdown"]}
        if mode == "blendenpik":
            passes = sum(i["lsqr_passes"] for i in infs)
            pass_ms = sum(i["ms_lsqr_pass"] for i in infs) / max(passes, 1)
            ent["lsqr_iters"] = infs[-1]["lsqr_iters"]
            ent["lsqr_pass_ms"] = pass_ms
            ent["lsqr_pass_gbs"] = 8.0 * n * (m + 2) / (pass_ms * 1e-3) / 1e9
            ent["cond_R"] = infs[-1]["cond_R"]
        out[mode] = ent
    if name == "c4":
        # the paper's cure for a numerically singular truncated basis (l.106,
        # l.395): Algorithm 2 with whitening, then Algorithm 1 (fab_basis_whiten)
        def solve_w(mode):
            sv.sketch(s, p.sketch_seed)
            sv.basis_whiten(m, k, 1000.0)
            sv.compress(mode, tol=1e-6)
            sv.apply(p.f, p.alpha, p.sigma, out=y)
            return sv.info()
        for mode in ("blendenpik", "sketch_solve", "none"):
            solve_w(mode)
            inf = solve_w(mode)
            t = inf["ms_sketch"] + inf["ms_basis"] + inf["ms_compress"] + inf["ms_apply"]
            ent = {"solves_per_s": 1e3 / t, "ms_per_solve": t, "ms_basis": inf["ms_basis"],
                   "ms_compress": inf["ms_compress"], "whitened_at": inf["whitened_at"],
                   "lsqr_iters": inf["lsqr_iters"], "cond_R": inf["cond_R"]}
            yw = y.cpu().numpy()
            ent["rel_diff_vs_unwhitened_blendenpik"] = float(np.linalg.norm(yw - res["blendenpik"][0]) /
                                                             np.linalg.norm(res["blendenpik"][0]))
            out["whitened_" + mode] = ent
    mb = min(i["ms_basis"] for i in res["blendenpik"][1])
    out["iters_per_s"] = m / (mb * 1e-3)
    out["basis_us_per_iter"] = mb * 1e3 / m
    out["basis_gbs"] = b_it * m / (mb * 1e-3) / 1e9
    fb = res["blendenpik"][0]
    nb = float(np.linalg.norm(fb))
    out["mode_agreement"] = {md: float(np.linalg.norm(res[md][0] - fb) / nb) for md in ("sketch_solve", "none")}
    out["f_m_finite"] = bool(all(np.isfinite(r[0]).all() for r in res.values()))
    sv.close()
    del sv, op, b, y
    torch.cuda.empty_cache()
    return out


def main():
    names = sys.argv[1:] or ["c1", "c2", "c4", "c3", "c5"]
    torch.cuda.set_device(0)
    for nm in names:
        try:
            r = run(nm)
        except Exception as e:     # report and continue with the next config
            r = {"config": nm, "error": repr(e)}
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()

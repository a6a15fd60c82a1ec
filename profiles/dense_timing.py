"""Device time of fab_apply's dense step f(alpha C + sigma I) e_1 (A6) at
m = 200 on c3-shaped matrices: fab_apply on a small-n c3 instance (g = 64,
n = 262144, so the combination K7 is ~0.07 ms of it) per function and per
sqrt algorithm (coupled Newton-Schulz, the default; Denman-Beavers under
FAB_DENSE_DB=1).  Prints one JSON line per case: ms_apply (median of 7),
dense_iters.

    python profiles/dense_timing.py > gpurun_out/dense_timing.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402


def run(g, m, f, alpha, sigma_rel, label):
    p = fp.make("c3", g=g, m=m, s=2 * m)
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
    sv.sketch(p.s, p.sketch_seed)
    sv.basis(p.m, p.k)
    sv.compress("sketch_solve")
    y = torch.empty(p.n, dtype=torch.float64, device="cuda")
    sigma = sigma_rel * p.norm_inf if sigma_rel else 0.0
    ts, its = [], []
    for _ in range(8):
        sv.apply(f, alpha, sigma, out=y)
        inf = sv.info()
        ts.append(inf["ms_apply"])
        its.append(inf["dense_iters"])
    sv.close()
    k7_ms = 8.0 * p.n * m / 6.5e12 * 1e3
    return {"case": label, "g": g, "n": p.n, "m": m, "f": f, "ms_apply": statistics.median(ts[1:]),
            "k7_model_ms": k7_ms, "dense_iters": its[-1]}


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for g in (64, 256):
        print(json.dumps(run(g, 200, "sqrt", 1.0, 1e-2, "sqrt " + os.environ.get("FAB_DENSE_DB", "ns"))), flush=True)
        print(json.dumps(run(g, 200, "exp", -1.0 / 12.0, 0.0, "exp")), flush=True)

"""Multi-RHS throughput (fab_basis_batch) on one B200:
Algorithm 2 (fused sketch) for p right-hand sides of one CSR operator, the
entries read once per Krylov step for all p vectors.

    python profiles/bench_multirhs.py > gpurun_out/multirhs.jsonl

c4 at its config (n = 2^22, m = 150, k = 2, s = 300); c5 at n = 2^25 with
m = 40 (V_{m+1} is 80.8 GB per right-hand side at m = 300, so p > 1 cannot
hold two bases on one GPU; the per-step cost does not depend on m for k = 2).
Reports Krylov iterations per second summed over the p right-hand sides.
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


def run(name, m, ps=(1, 2, 4), reps=3, env=None, tag=None):
    """env: FAB_* variables set for this run only (plan widths are read when
    a context / batch plan is built)."""
    saved = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        _run(name, m, ps, reps, tag or name, env or {})
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _run(name, m, ps, reps, tag, env):
    t0 = time.perf_counter()
    p = fp.make(name, m=m, s=2 * m)
    print(f"[{name}] generated in {time.perf_counter() - t0:.1f} s", file=sys.stderr, flush=True)
    op = fab.Operator.from_problem(p)
    res = {"config": name, "tag": tag, "env": env, "n": p.n, "m": m, "k": p.k, "s": p.s, "nnz": int(p.meta.get("nnz", 0))}
    for nb in ps:
        svs = []
        for i in range(nb):
            b = p.b if i == 0 else np.random.default_rng(7000 + i).standard_normal(p.n)
            svs.append(fab.Solver(op, torch.as_tensor(b).cuda(), m, p.k, p.s))
        ts = []
        for r in range(reps + 1):
            for sv in svs:
                sv.sketch(p.s, p.sketch_seed)
            if nb == 1:
                svs[0].basis(m, p.k)
            else:
                fab.basis_batch(svs, m, p.k)
            if r:
                ts.append(svs[0].info()["ms_basis"])
        ms = statistics.median(ts)
        res[f"p{nb}"] = {"ms_basis": ms, "iters_per_s_total": nb * m / (ms * 1e-3),
                         "us_per_step_per_rhs": ms * 1e3 / (m * nb)}
        for sv in svs:
            sv.close()
        del svs
        torch.cuda.empty_cache()
    print(json.dumps(res), flush=True)


def main():
    torch.cuda.set_device(0)
    which = sys.argv[1:] or ["c4", "c4_cb1", "c4_cb2", "c5"]
    for w in which:
        if w == "c4":        # batch plan by the L2 rule (p = 4: 3 column blocks of the interleaved copy)
            run("c4", 150)
        elif w == "c4_cb1":  # the single-RHS plan column-blocked too (2 blocks of 2^21 columns)
            run("c4", 150, ps=(1,), env={"FAB_CSR_COLBLOCK": str(1 << 21)}, tag="c4_colblock2")
        elif w == "c4_cb2":  # p = 2 / 4 with narrower batch blocks
            run("c4", 150, ps=(2, 4), env={"FAB_BATCH_COLBLOCK": str(1 << 20)}, tag="c4_batchblock_2^20")
        elif w == "c5":
            run("c5", 40)


if __name__ == "__main__":
    main()

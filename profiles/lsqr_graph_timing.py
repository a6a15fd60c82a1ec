"""Solve latency with the host-driven LSQR loop (FAB_LSQR_GRAPH=0: a host
poll every 4 iterations, one launch per kernel) against the graph-resident
loop (one CUDA graph, conditional WHILE node, the tolerance test on the
device), and the graph loop with FAB_FLAG_ASYNC (fab_basis / fab_compress
enqueue only; fab_apply resolves), at the small BASELINE configs where latency matters (c1, c2) and at
c3 for reference.  Blendenpik-LSQR tol 1e-6, fused sketch, A and b resident.

    python profiles/lsqr_graph_timing.py > gpurun_out/lsqr_graph.jsonl

Per config and loop: median over `reps` solves of the wall time of the five
ABI calls (host clock around a synchronised solve: the latency a caller
sees) and of fab_compress's own device time (CUDA events, fab_info).
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402


def run(name, reps, **kw):
    p = fp.make(name, **kw)
    y = torch.empty(p.n, dtype=torch.float64, device="cuda")
    out = {"config": name, "n": p.n, "m": p.m}
    for flag in ("0", "1", "async"):
        # host loop / graph loop (synchronous calls) / graph loop with
        # FAB_FLAG_ASYNC (fab_basis and fab_compress only enqueue)
        os.environ["FAB_LSQR_GRAPH"] = "0" if flag == "0" else "1"
        sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s,
                        asynchronous=(flag == "async"))
        walls, comp = [], []
        for i in range(reps + 3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sv.sketch(p.s, p.sketch_seed)
            sv.basis(p.m, p.k)
            sv.compress("blendenpik", tol=1e-6)
            sv.apply(p.f, p.alpha, p.sigma, out=y)
            torch.cuda.synchronize()
            if i >= 3:
                walls.append((time.perf_counter() - t0) * 1e6)
                comp.append(sv.info()["ms_compress"] * 1e3)
        key = {"0": "host_loop", "1": "graph", "async": "graph_async"}[flag]
        out[key] = {"us_per_solve": statistics.median(walls), "compress_us": statistics.median(comp),
                    "lsqr_iters": sv.info()["lsqr_iters"]}
        sv.close()
    return out


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for name, reps in (("c1", 200), ("c2", 50), ("c3", 5)):
        print(json.dumps(run(name, reps)), flush=True)

"""K5 (the batched SRHT of V_{m+1}, API order: sketch drawn after the basis)
A/B: k_sketch_direct (default), the tile-group kernel k_sketch_groups
(FAB_SKETCH_K5=2) and the warp sub-tile kernel k_sketch_warp (=3), at BASELINE c3 (n = 2^24, m = 200: 8 n (m+1) = 27.0 GB
per pass) and c2.  Prints per kernel the pass time (CUDA events, fab_info
ms_sketch_batched, median of 5), its GB/s against the algorithmic bytes, and
whether Theta V is bitwise equal to the fused (K3) sketch (else its max
relative difference).

    python profiles/k5_ab.py > gpurun_out/k5_ab.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402


def run(name, **kw):
    p = fp.make(name, **kw)
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
    sv.sketch(p.s, p.sketch_seed)
    sv.basis(p.m, p.k)                 # fused: Theta V from K3
    fused = sv.get("SV")
    out = {"config": name, "n": p.n, "m": p.m, "s": p.s, "bytes": 8.0 * p.n * (p.m + 1)}
    for label, env in (("k_sketch_warp", "3"), ("k_sketch_direct", "1"), ("k_sketch_groups", "2")):
        os.environ["FAB_SKETCH_K5"] = env
        ts = []
        for _ in range(6):
            sv.basis(p.m, p.k)
            sv.sketch(p.s, p.sketch_seed)
            sv.compress("sketch_solve")
            ts.append(sv.info()["ms_sketch_batched"])
        ms = statistics.median(ts[1:])
        out[label] = {"ms": ms, "gbs": out["bytes"] / (ms * 1e-3) / 1e9,
                      "bitwise_equal_fused": bool(np.array_equal(sv.get("SV"), fused)),
                      "maxrel_vs_fused": float(np.abs(sv.get("SV") - fused).max() / np.abs(fused).max())}
    sv.close()
    return out


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for name, kw in (("c2", {}), ("c3", {})):
        print(json.dumps(run(name, **kw)), flush=True)

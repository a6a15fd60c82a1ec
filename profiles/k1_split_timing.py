"""Single-GPU cost of the multi-GPU K1 split: one rank's
z-slab of c3 at P = 2, 4, 8 (256 x 256 x 256/P planes of the c3 stencil) as
a standalone operator, Algorithm 2 steps (K1 + K3, fused sketch) timed with
the whole-block K1 and with FAB_FORCE_K1_SPLIT=1 (K1 as interior rows +
boundary slabs, the launch structure the ranks use while the halo is in
flight; here the side stream sends nothing).  The difference is what the
overlap costs; the halo it hides is one 512-KB plane per neighbour.

    python profiles/k1_split_timing.py > gpurun_out/k1_split.jsonl
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


def run(P, m=50, reps=5):
    g = 256
    coeffs, _ = fp.stencil_coeffs(3, g)
    dims = (g, g, g // P)
    n = g * g * (g // P)
    b = np.random.default_rng(P).standard_normal(n)
    out = {"P": P, "rows_per_rank": n, "m": m}
    for flag in ("0", "1"):
        os.environ["FAB_FORCE_K1_SPLIT"] = flag
        sv = fab.Solver(fab.Operator.stencil(dims, coeffs), torch.as_tensor(b).cuda(), m, 4, 400)
        ts = []
        for i in range(reps + 1):
            sv.sketch(400, 3003)
            sv.basis(m, 4)
            if i:
                ts.append(sv.info()["ms_basis"])
        H = sv.get("H")
        sv.close()
        key = "split" if flag == "1" else "whole"
        out[key] = {"us_per_step": statistics.median(ts) * 1e3 / m}
        out[key + "_H"] = H
    out["H_rel_diff"] = float(np.linalg.norm(out["split_H"] - out["whole_H"]) / np.linalg.norm(out["whole_H"]))
    del out["split_H"], out["whole_H"]
    os.environ["FAB_FORCE_K1_SPLIT"] = "0"
    return out


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for P in (2, 4, 8):
        print(json.dumps(run(P)), flush=True)

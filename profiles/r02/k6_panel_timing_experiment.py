"""Timing experiment for a panel-blocked V: the K6 pass of
c3 (n = 2^24, m = 200) reading the same memory as row panels of P rows x
(m_max+1) columns through a 3-D tensor map (FAB_K6_PANEL=P; the values are
not V's -- only the access pattern is), against the column-major layout.

    python profiles/k6_panel_timing.py > gpurun_out/k6_panel.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402

torch.cuda.set_device(0)
p = fp.make("c3")
sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s, profile=True)
sv.sketch(p.s, p.sketch_seed)
sv.basis(p.m, p.k)
for panel in ("0", "512", "2048", "8192", "65536", "0"):
    os.environ["FAB_K6_PANEL"] = panel
    best = 0.0
    for _ in range(3):
        sv.compress("blendenpik", iters=20)
        inf = sv.info()
        gbs = 8.0 * p.n * (p.m + 2) * inf["lsqr_passes"] / (inf["ms_lsqr_pass"] * 1e-3) / 1e9
        best = max(best, gbs)
    print(json.dumps({"panel_rows": int(panel), "k6_gbs": best}), flush=True)
sv.close()

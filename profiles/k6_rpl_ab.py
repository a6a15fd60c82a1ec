"""A/B of K6 (k_lsqr_pipe) box height: rows per lane RPL (box = 32 RPL rows)
and KEEP (chunk kept in registers vs re-read from shared memory), selected
per process by FAB_LSQR_RPL / FAB_LSQR_KEEP.  Config c3 (n = 2^24, m = 200)
by default, or c2 / c5 shapes; one process per variant.

    python profiles/k6_rpl_ab.py c3 rpl1:FAB_LSQR_RPL=1 rpl2:FAB_LSQR_RPL=2 ...
prints per variant: ms per LSQR pass (CUDA events, FAB_FLAG_PROFILE), its
bytes 8n(m+2) / time, compress ms, iterations, and a hash of f_m.
"""
import hashlib
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(name):
    import numpy as np
    import torch
    import fab_problems as fp
    import paper_2212_12758_b200 as fab
    torch.cuda.set_device(0)
    p = fp.make(name)
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s, profile=True)
    y = torch.empty(p.n, dtype=torch.float64, device="cuda")
    res = []
    for r in range(4):
        sv.sketch(p.s, p.sketch_seed)
        sv.basis(p.m, p.k)
        sv.compress("blendenpik", tol=1e-6)
        sv.apply(p.f, p.alpha, p.sigma, out=y)
        inf = sv.info()
        if r:
            res.append(inf)
    fm = y.cpu().numpy()
    pm = statistics.median(i["ms_lsqr_pass"] for i in res)
    return dict(ms_lsqr_pass=pm, pass_gbs=8.0 * p.n * (p.m + 2) / (pm * 1e-3) / 1e9,
                ms_compress=statistics.median(i["ms_compress"] for i in res),
                lsqr_iters=res[-1]["lsqr_iters"], fm_sha=hashlib.sha256(fm.tobytes()).hexdigest()[:16],
                fm_norm=float(np.linalg.norm(fm)))


def main():
    if sys.argv[1] == "--child":
        print(json.dumps(child(sys.argv[2])))
        return
    name = sys.argv[1]
    for spec in sys.argv[2:]:
        tag, _, envs = spec.partition(":")
        extra = dict(kv.split("=", 1) for kv in envs.split(",")) if envs else {}
        env = dict(os.environ)
        env.update(extra)
        r = subprocess.run([sys.executable, __file__, "--child", name], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 and r.stdout.strip() else None
        res = json.loads(line) if line else dict(error=r.stderr[-800:])
        res.update(config=name, variant=tag, env=extra)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

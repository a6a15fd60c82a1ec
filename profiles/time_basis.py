"""Time fab_basis alone (fused sketch) on the c3 workload: python profiles/time_basis.py [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = fp.make("c3")
sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
ts = []
for i in range(reps + 1):
    sv.sketch(p.s, p.sketch_seed)
    sv.basis(p.m, p.k)
    if i:
        ts.append(sv.info()["ms_basis"])
ms = min(ts)
print(f"basis ms min {ms:.2f} (all {['%.2f' % t for t in ts]}) it/s {p.m / ms * 1e3:.0f} "
      f"env MF={os.environ.get('FAB_MATRIX_FREE')} DBG={os.environ.get('FAB_MF_DEBUG')}")

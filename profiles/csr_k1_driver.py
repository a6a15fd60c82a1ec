"""Driver for ncu captures of the CSR K1 (k_csr_stream): Algorithm 2 on
config NAME (c4 or c5) with P right-hand sides (P = 1: fab_basis; P > 1:
fab_basis_batch, one entry stream for all P vectors).

    ncu ... -k regex:k_csr_stream python profiles/csr_k1_driver.py c4 2
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
m = 8
p = fp.make(name, m=m, s=2 * m)
op = fab.Operator.from_problem(p)
svs = [fab.Solver(op, torch.as_tensor(p.b if i == 0 else np.random.default_rng(7000 + i).standard_normal(p.n)).cuda(),
                  m, p.k, p.s) for i in range(P)]
for sv in svs:
    sv.sketch(p.s, p.sketch_seed)
if P == 1:
    svs[0].basis(m, p.k)
else:
    fab.basis_batch(svs, m, p.k)
torch.cuda.synchronize()
print(name, P, svs[0].info()["ms_basis"], file=sys.stderr)

"""Algorithm 1 (sketched Gram-Schmidt) basis on c3 (argv[1] = m) and, with a
second argument, the full Arnoldi (CGS2) basis: the tall GEMVs K6n / K6.
Driver for the K6n ncu capture in profiles/run_profiles.sh."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import fab_problems as fp, paper_2212_12758_b200 as fab
m = int(sys.argv[1]) if len(sys.argv) > 1 else 200
p = fp.make("c3", m=m)
sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
sv.sketch(p.s, p.sketch_seed)
for i in range(2):
    sv.basis_sgs(p.m)
    print("sgs basis ms", sv.info()["ms_basis"], file=sys.stderr)
if len(sys.argv) > 2:
    for i in range(2):
        sv.basis_arnoldi(p.m)
        print("arnoldi basis ms", sv.info()["ms_basis"], file=sys.stderr)

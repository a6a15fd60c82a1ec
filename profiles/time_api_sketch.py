"""API-order sketch (K5, k_sketch_direct) on c3 with m columns: basis first, then
fab_sketch, then a compress that needs Theta V (sketch-and-solve).  Driver for
the K5 ncu capture in profiles/run_profiles.sh."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import fab_problems as fp, paper_2212_12758_b200 as fab
m = int(sys.argv[1]) if len(sys.argv) > 1 else 40
p = fp.make("c3", m=m)
sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
for i in range(3):
    sv.basis(p.m, p.k)
    sv.sketch(p.s, p.sketch_seed)
    sv.compress("sketch_solve")
    print("api sketch ms", sv.info()["ms_sketch_batched"], file=sys.stderr)

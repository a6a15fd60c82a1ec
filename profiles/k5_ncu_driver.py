"""ncu driver for K5 (the batched SRHT after the basis) at BASELINE c3: one
API-order solve (basis, then sketch, then sketch-and-solve), so the only K5
launch is the batched pass over V_{m+1} (the fused prologue is not taken).

    ncu --set full -k regex:k_sketch_warp -c 1 python profiles/k5_ncu_driver.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402

if __name__ == "__main__":
    torch.cuda.set_device(0)
    p = fp.make(sys.argv[1] if len(sys.argv) > 1 else "c3")
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
    sv.basis(p.m, p.k)
    sv.sketch(p.s, p.sketch_seed)
    sv.compress("sketch_solve")
    print("ms_sketch_batched", sv.info()["ms_sketch_batched"])
    sv.close()

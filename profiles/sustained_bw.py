"""Sustained bandwidth under the power cap: a 2 GiB torch copy and read loop
(4 s each) next to the fused LSQR pass K6 (c3, fixed 40 iterations, 6 s),
with the SM clock / power nvidia-smi reports at the end of each loop."""
import sys, os, time, subprocess, json
sys.path.insert(0, os.getcwd())
import torch
import fab_problems as fp, paper_2212_12758_b200 as fab
dev = torch.device("cuda:0")
def clocks():
    o = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw", "--format=csv,noheader,nounits"],
                       capture_output=True, text=True).stdout.strip()
    return o
N = 1 << 28   # 2 GiB fp64
a = torch.empty(N, dtype=torch.float64, device=dev).normal_()
b = torch.empty_like(a)
def time_loop(fn, bytes_per, secs):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 0; t_end = time.time() + secs; k = 0; tot = 0.0; cl = []
    while time.time() < t_end:
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1); gbs = bytes_per / ms / 1e6
        best = max(best, gbs); tot += gbs; k += 1
        if k % 20 == 0: cl.append(clocks())
    return best, tot / k, cl[-1] if cl else clocks()
out = {}
out["copy_burst_first"] = time_loop(lambda: b.copy_(a), 2 * 8 * N, 0.5)
out["copy_sustained"] = time_loop(lambda: b.copy_(a), 2 * 8 * N, 4.0)
out["read_sustained"] = time_loop(lambda: a.sum(), 8 * N, 4.0)
del a, b
torch.cuda.empty_cache()
p = fp.make("c3")
sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s, profile=True)
sv.sketch(p.s, p.sketch_seed); sv.basis(p.m, p.k)
res = []
t_end = time.time() + 6
while time.time() < t_end:
    sv.compress("blendenpik", iters=40)
    inf = sv.info(); res.append(8.0 * p.n * (p.m + 2) / (inf["ms_lsqr_pass"] / max(inf["lsqr_passes"], 1) * 1e-3) / 1e9)
out["lsqr_pass_gbs_sustained"] = (max(res), sum(res) / len(res), clocks())
print(json.dumps(out))

"""SM clock and board power while K5 (the batched SRHT pass, FP64 butterflies +
HBM stream) runs back to back, against K6-dominated Blendenpik compressions,
at BASELINE c3.  nvidia-smi is polled every 100 ms in a side process.

    python profiles/k5_clocks.py > gpurun_out/k5_clocks.jsonl
"""
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fab_problems as fp  # noqa: E402
import paper_2212_12758_b200 as fab  # noqa: E402


def sampled(fn, seconds):
    q = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "100", "-i", "0"],
                         stdout=subprocess.PIPE, text=True)
    t0 = time.perf_counter()
    reps, extra = 0, []
    while time.perf_counter() - t0 < seconds:
        extra.append(fn())
        reps += 1
    torch.cuda.synchronize()
    q.terminate()
    rows = [l.split(", ") for l in q.communicate()[0].strip().splitlines()]
    rows = rows[len(rows) // 3:]            # the loaded part
    return {"reps": reps, "sm_mhz_median": statistics.median(float(r[0]) for r in rows),
            "sm_mhz_min": min(float(r[0]) for r in rows),
            "power_w_median": statistics.median(float(r[1]) for r in rows),
            "reasons": sorted({r[2] for r in rows}), "samples": len(rows),
            "ms_median": statistics.median(e for e in extra if e is not None) if any(e is not None for e in extra) else None}


def main():
    torch.cuda.set_device(0)
    p = fp.make("c3")
    sv = fab.Solver(fab.Operator.from_problem(p), torch.as_tensor(p.b).cuda(), p.m, p.k, p.s)
    sv.sketch(p.s, p.sketch_seed)
    sv.basis(p.m, p.k)

    def k5():
        sv.sketch(p.s, p.sketch_seed)          # marks Theta V stale: compress runs the batched K5
        sv.compress("sketch_solve")
        return sv.info()["ms_sketch_batched"]

    def k6():
        sv.compress("blendenpik")
        return sv.info()["ms_compress"]

    for label, fn in (("k5_loop", k5), ("k6_loop", k6), ("k5_loop_again", k5)):
        out = sampled(fn, 6.0)
        out["loop"] = label
        print(json.dumps(out), flush=True)
    sv.close()


if __name__ == "__main__":
    main()

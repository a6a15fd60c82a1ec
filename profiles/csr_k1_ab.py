"""A/B timing of the CSR basis (K1 + K3 per Krylov step) across library
variants (profiles/build_variant.py): one process per variant, the c4 / c5
problem generated once and kept in /tmp as .npy (seeded: the same arrays).

    python profiles/csr_k1_ab.py c4 150 base:profiles/variants/libfab_base.so pre6:...
    spec = TAG:LIB[:P[:ENV=VAL,ENV=VAL]]   (LIB "default" = the in-tree build;
    P right-hand sides through fab_basis_batch, default 1)
prints one JSON line per variant: median ms per basis and us per step (per
right-hand side).
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cache(name):
    d = f"/tmp/fab_ab_{name}"
    if not os.path.exists(os.path.join(d, "done")):
        import numpy as np
        import fab_problems as fp
        p = fp.make(name)
        os.makedirs(d, exist_ok=True)
        ip, ix, dv = p._csr
        for k, v in dict(ip=ip, ix=ix, dv=dv, b=p.b).items():
            np.save(os.path.join(d, k + ".npy"), v)
        open(os.path.join(d, "done"), "w").write("1")
    return d


def child(name, m, nrhs=1, reps=5):
    import numpy as np
    import torch
    import paper_2212_12758_b200 as fab
    d = cache(name)
    ip, ix, dv, b = (np.load(os.path.join(d, k + ".npy")) for k in ("ip", "ix", "dv", "b"))
    torch.cuda.set_device(0)
    op = fab.Operator.csr(ip, ix, dv)
    k, s = 2, 2 * m
    svs = [fab.Solver(op, torch.as_tensor(b if i == 0 else np.random.default_rng(7000 + i).standard_normal(len(b)))
                      .cuda(), m, k, s) for i in range(nrhs)]
    ts = []
    for r in range(reps + 1):
        for sv in svs:
            sv.sketch(s, 3004)
        if nrhs == 1:
            svs[0].basis(m, k)
        else:
            fab.basis_batch(svs, m, k)
        if r:
            ts.append(svs[0].info()["ms_basis"])
    ms = statistics.median(ts)
    import hashlib
    hsh = hashlib.sha256(np.ascontiguousarray(svs[0].get("H")).tobytes()).hexdigest()[:16]
    return dict(ms_basis=ms, p=nrhs, us_per_step_per_rhs=1e3 * ms / (m * nrhs), all=ts, H_sha=hsh)


def main():
    if sys.argv[1] == "--child":
        print(json.dumps(child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))))
        return
    name, m = sys.argv[1], int(sys.argv[2])
    cache(name)
    for spec in sys.argv[3:]:
        parts = spec.split(":")
        tag, lib = parts[0], parts[1]
        nrhs = int(parts[2]) if len(parts) > 2 else 1
        extra = dict(kv.split("=", 1) for kv in parts[3].split(",")) if len(parts) > 3 and parts[3] else {}
        env = dict(os.environ)
        env.update(extra)
        if lib != "default":
            env["FAB_LIB_VARIANT"] = os.path.abspath(lib)
        r = subprocess.run([sys.executable, __file__, "--child", name, str(m), str(nrhs)], env=env,
                           capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 and r.stdout.strip() else None
        res = json.loads(line) if line else dict(error=r.stderr[-500:])
        res.update(config=name, m=m, variant=tag, env=extra)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

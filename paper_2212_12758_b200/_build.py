"""In-tree build of libfab.so (sm_100a) with nvcc.

    python paper_2212_12758_b200/_build.py [--force] [--ptxas-v]

Every .cu under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17
and linked into paper_2212_12758_b200/libfab.so (static cudart).  The .so is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
OUT = os.path.join(HERE, "libfab.so")
OBJ = os.path.join(HERE, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
def nccl_include():
    """nccl.h of the NCCL that torch ships (libnccl.so.2 is dlopen'ed at run time)."""
    try:
        import nvidia.nccl
        for base in list(getattr(nvidia.nccl, "__path__", [])):
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except ImportError:
        pass
    for inc in ("/usr/include", "/usr/local/include"):
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel or system NCCL headers)")


FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                "--expt-relaxed-constexpr", "-I", INC, "-I", nccl_include()]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(INC, "fab.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, ptxas_verbose=False, quiet=False):
    os.makedirs(OBJ, exist_ok=True)
    nv = nvcc()
    hdr = headers()
    jobs = []
    objs = []
    for src in sources():
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdr):
            cmd = [nv] + FLAGS + (["-Xptxas", "-v"] if ptxas_verbose else []) + ["-c", src, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    failed = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for cmd, r in ex.map(run, jobs):
            if r.returncode != 0:
                failed.append((cmd, r.stderr))
            elif (ptxas_verbose or r.stderr.strip()) and not quiet:
                sys.stderr.write(r.stderr)
    if failed:
        msg = "\n".join(" ".join(c) + "\n" + e for c, e in failed)
        raise RuntimeError("nvcc failed:\n" + msg)
    if force or jobs or _stale(OUT, objs):
        cmd = [nv] + ARCH + ["-shared", "-o", OUT] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, ptxas_verbose="--ptxas-v" in sys.argv))

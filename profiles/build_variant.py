"""Profiling A/B: build a variant of libfab.so with extra -D flags on some
sources (the other objects are the in-tree build's), into
profiles/variants/libfab_<tag>.so (git-ignored).  Load it in a measurement
script with FAB_LIB_VARIANT=<path>.

    python profiles/build_variant.py TAG csr.cu -DFAB_CSR_OCC=5 [-DX=Y ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2212_12758_b200"))
import _build as B  # noqa: E402


def main():
    tag, srcs, defs = sys.argv[1], [a for a in sys.argv[2:] if a.endswith(".cu")], \
        [a for a in sys.argv[2:] if a.startswith("-D")]
    B.build(quiet=True)
    out_dir = os.path.join(ROOT, "profiles", "variants", tag)
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    for src in B.sources():
        base = os.path.basename(src)
        if base in srcs:
            obj = os.path.join(out_dir, base[:-3] + ".o")
            subprocess.run([B.nvcc()] + B.FLAGS + defs + ["-c", src, "-o", obj], check=True)
        else:
            obj = os.path.join(B.OBJ, base[:-3] + ".o")
        objs.append(obj)
    out = os.path.join(ROOT, "profiles", "variants", f"libfab_{tag}.so")
    subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", out] + objs + ["-ldl"], check=True)
    print(out)


if __name__ == "__main__":
    main()

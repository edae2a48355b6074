"""Build the in-tree CUDA library libras_b200.so for sm_100a (nvcc, no JIT cache).

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libras_b200.so")
SOURCES = ["plan.cpp", "factor.cpp", "zformat.cpp", "solver.cu", "async.cu"]


def nccl_dir() -> str:
    import nvidia.nccl  # torch's bundled NCCL (same libnccl.so.2 torch loads)

    return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    OUT_ = out
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs += [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    if not force and os.path.exists(OUT_):
        t = os.path.getmtime(OUT_)
        if all(os.path.getmtime(f) <= t for f in srcs + hdrs):
            return OUT_
    nd = nccl_dir()
    cmd = [
        "nvcc", "-O3", "-std=c++17", "-lineinfo",
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-Xcompiler", "-fPIC,-O3", "-shared",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nd, "include"),
        "-Xptxas", "-v" if verbose else "-O3",
        *["-D" + d for d in defines],
        "-o", OUT_ + ".tmp", *srcs,
        "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
        "-Xlinker", "-rpath=" + os.path.join(nd, "lib"),
    ]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libras_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(OUT_ + ".tmp", OUT_)
    return OUT_


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out PATH] [-DNAME=VAL ...]  (variants for tuning sweeps)
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else OUT
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args or bool(defs), verbose="-v" in args, out=out, defines=defs))

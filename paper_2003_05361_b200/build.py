"""Build the in-tree CUDA library libras_b200.so for sm_100a (nvcc, no JIT cache).

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
Provenance: the build stamps a hash of every source, header, define and flag
into the library (`ras_build_hash()`); the binding (`_ffi.lib()`) recomputes
it from the tree and refuses to load a library built from other sources, and
`__graft_entry__.build()` always recompiles.  Translation units compile in
parallel (one nvcc per source), then link.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libras_b200.so")
SOURCES = ["plan.cpp", "factor.cpp", "zformat.cpp", "comm.cu", "setup_dev.cu", "solver.cu", "async.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-O3"]


def nccl_dir() -> str:
    import nvidia.nccl  # torch's bundled NCCL (same libnccl.so.2 torch loads)

    return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]


def _inputs():
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    hdrs = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh")))
    inc = os.path.join(ROOT, "include")
    hdrs += sorted(os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h"))
    return srcs, hdrs


def source_hash(defines=()) -> str:
    """sha256 over the sources, headers, defines and compiler flags (16 hex digits)."""
    h = hashlib.sha256()
    srcs, hdrs = _inputs()
    for f in srcs + hdrs:
        h.update(os.path.relpath(f, ROOT).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(repr((list(defines), FLAGS)).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    OUT_ = out
    srcs, hdrs = _inputs()
    hsh = source_hash(defines)
    if not force and os.path.exists(OUT_) and os.path.exists(OUT_ + ".hash"):
        with open(OUT_ + ".hash") as fh:
            if fh.read().strip() == hsh:
                return OUT_
    nd = nccl_dir()
    objdir = os.path.join(ROOT, "build", "obj_" + hashlib.sha1(OUT_.encode()).hexdigest()[:8])
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nd, "include")]
    defs = ["-D" + d for d in defines] + [f"-DRAS_BUILD_HASH=\"{hsh}\""]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = ["nvcc", *FLAGS, *inc, "-Xptxas", "-v" if verbose else "-O3", *defs, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return obj, r

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, srcs))
    for (obj, r), src in zip(results, srcs):
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)} building libras_b200.so")
        if verbose:
            sys.stderr.write(r.stderr)
    link = ["nvcc", *ARCH, "-shared", "-o", OUT_ + ".tmp", *[o for o, _ in results],
            "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed building libras_b200.so")
    os.replace(OUT_ + ".tmp", OUT_)
    with open(OUT_ + ".hash", "w") as fh:
        fh.write(hsh + "\n")
    return OUT_


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out PATH] [-DNAME=VAL ...]  (variants for tuning sweeps)
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else OUT
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args or bool(defs), verbose="-v" in args, out=out, defines=defs))

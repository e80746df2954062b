"""Build the in-tree CUDA library ``librcg.so`` for sm_100a with nvcc.

The library is built in-tree (``paper_1301_7530_b200/librcg.so``) so it travels
to the GPU box with the repo snapshot; nothing is JIT-compiled at import time.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "librcg.so"
SOURCES = ["api.cu", "spmv.cu", "dense.cu", "pcg.cu", "ritz.cu", "comm.cu", "vmm.cu", "gen.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def needs_rebuild():
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "rcg.h"]
    return any(p.exists() and p.stat().st_mtime > t for p in deps)


def build(force=False, verbose=True, extra=()):
    """One nvcc per translation unit, in parallel (objects under build/), then
    one shared-library link."""
    if not force and not needs_rebuild():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    obj_dir = PKG.parent / "build" / "obj"
    obj_dir.mkdir(parents=True, exist_ok=True)
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v" if os.environ.get("RCG_PTXAS_VERBOSE") else "-O3",
              "-I", str(PKG.parent / "include"), *extra]

    def compile_one(src):
        obj = obj_dir / (Path(src).stem + ".o")
        cmd = [*common, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return str(obj)

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    link = [nvcc(), *ARCH, "-shared", "-o", str(LIB) + ".tmp", *objs, "-ldl"]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)

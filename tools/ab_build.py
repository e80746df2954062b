"""Build librcg.so variants for on-box A/B runs (RCG_LIB=<path> selects one).

usage: python tools/ab_build.py NAME [-DFLAG=V ...] [--src DIR]
Writes paper_1301_7530_b200/ab/NAME/librcg.so (git-ignored, travels to the box).
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
from paper_1301_7530_b200 import _build  # noqa: E402

name = sys.argv[1]
args = sys.argv[2:]
src = REPO / "paper_1301_7530_b200" / "csrc"
if "--src" in args:
    i = args.index("--src")
    src = Path(args[i + 1])
    del args[i:i + 2]
out = REPO / "paper_1301_7530_b200" / "ab" / name
obj = out / "obj"
obj.mkdir(parents=True, exist_ok=True)
common = [_build.nvcc(), *_build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
          "-I", str(REPO / "include"), *args]


def one(s):
    o = obj / (Path(s).stem + ".o")
    subprocess.run([*common, "-c", str(src / s), "-o", str(o)], check=True)
    return str(o)


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, _build.SOURCES))
subprocess.run([_build.nvcc(), *_build.ARCH, "-shared", "-o", str(out / "librcg.so"), *objs, "-ldl"], check=True)
print(out / "librcg.so")

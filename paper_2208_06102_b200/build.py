"""Builds the CUDA library in-tree: paper_2208_06102_b200/libzeus_sim.so (sm_100a).

NC-1: --fmad=false so no multiply-add is contracted behind the contract's back;
fp64 division and sqrt are IEEE round-to-nearest by default.
"""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libzeus_sim.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
    "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh"))
                  + [os.path.join(ROOT, "include", "zeus_sim.h")])


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=(), extra=()) -> str:
    """Compiles csrc/zeus_sim.cu into ``out``; ``defines`` (e.g. ["ZS_PAIR_UNROLL=2"]) are
    for kernel A/B builds only."""
    srcs = sources()
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(f) for f in srcs):
        return out
    tmp = f"{out}.tmp{os.getpid()}"                 # written aside, then renamed into place, so a
    cmd = [NVCC, *FLAGS, *extra, *[f"-D{d}" for d in defines], "-o", tmp,   # concurrent loader
           os.path.join(HERE, "csrc", "zeus_sim.cu"), "-lcudart"]          # never sees half a file
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    os.replace(tmp, out)
    with open(out + ".ptxas.log", "w") as f:
        f.write(r.stderr)
    if verbose:
        print(r.stderr)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))

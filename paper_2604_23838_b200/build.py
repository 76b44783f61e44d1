"""Build the in-tree CUDA library `librlx.so` for sm_100a.

    python -m paper_2604_23838_b200.build [--verbose]

The library is the only scoring path (no CPU fallback). It is compiled
with -fmad=false so that no multiply-add is contracted: every double
expression rounds exactly like the reference's Python floats.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librlx.so")
SOURCES = ("rlx_abi.cu", "rlx_kernels.cu", "rlx_plan.cpp", "rlx_state.cpp", "rlx_graph.cu", "rlx_sim.cpp", "rlx_bnb.cpp")
HEADERS = ("rlx_plan.hpp", "rlx_hostplan.hpp", "rlx_state.hpp")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale(lib: str = None) -> bool:
    lib = lib or LIB
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "rlx.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: tuple = ()) -> str:
    """Compile librlx.so. `out`/`defines` build a side variant (tuning
    experiments, e.g. -DRLX_T2=640); the product is always LIB."""
    lib = out or LIB
    if not force and not _stale(lib):
        return lib
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src + ".o")
        cmd = [nvcc(), ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-ffp-contract=off", "-c", os.path.join(CSRC, src), "-o", obj]
        for d in defines:
            cmd.insert(1, "-D" + d)
        if out or defines:
            obj = obj + "." + os.path.basename(lib) + ".o"
            cmd[-1] = obj
        if verbose and src.endswith("kernels.cu"):
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = lib + ".tmp"
    subprocess.run([nvcc(), ARCH, "-shared", "-o", tmp, *objs, "-lcudart"], check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out = next((a.split("=", 1)[1] for a in args if a.startswith("--out=")), None)
    defs = tuple(a[2:] for a in args if a.startswith("-D"))
    print(build(force=True, verbose="--verbose" in args, out=out, defines=defs))

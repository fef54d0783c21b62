"""Build the in-tree CUDA library ``libconvgemm_b200.so`` for sm_100a.

Plain ``nvcc -shared`` over ``csrc/*.cu`` (no torch types in any signature), so the
C-ABI in ``include/convgemm_b200.h`` is exactly what a non-Python host would link.
The ``.so`` lands next to this file, is git-ignored, and travels to the GPU box
with the repository snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libconvgemm_b200.so")
# profiling variant for tools/ (CGB_* environment knobs, CGB_DEBUG_SW stage switches and
# per-CTA counters); never loaded by the package unless CGB_LIB_OVERRIDE points at it
LIB_PROF = os.path.join(HERE, "libconvgemm_b200_prof.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps.append(os.path.join(os.path.dirname(HERE), "include", "convgemm_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, profiling: bool = False) -> str:
    lib = LIB_PROF if profiling else LIB
    if not force and not stale(lib):
        return lib
    tmp = lib + ".tmp"
    extra = ["-DCGB_PROFILING"] if profiling else []
    # one nvcc per translation unit in parallel (the shifted-window kernel instantiates
    # ~50 configurations), then one device-aware link
    objdir = os.path.join(HERE, "build", "prof" if profiling else "rel")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in FLAGS if f != "-shared"]

    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    hdrs.append(os.path.join(os.path.dirname(HERE), "include", "convgemm_b200.h"))
    hdrs.append(os.path.abspath(__file__))

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        # objects are reused while newer than their source and every header
        if not force and os.path.exists(obj) and all(
                os.path.getmtime(d) < os.path.getmtime(obj) for d in [src, *hdrs] if os.path.exists(d)):
            return obj
        cmd = [NVCC, *compile_flags, *extra, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(sources())) as ex:
        objs = list(ex.map(compile_one, sources()))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", tmp]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, profiling="--profiling" in sys.argv))

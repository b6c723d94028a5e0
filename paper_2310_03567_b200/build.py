"""In-tree build of the CUDA library ``_lodb200.so`` (sm_100a only).

``python -m paper_2310_03567_b200.build`` (or ``__graft_entry__.build()``)
compiles csrc/*.cu with nvcc straight into the package directory, so the
shared object travels with the repo snapshot to the GPU box.  Flags:

* ``-gencode arch=compute_100a,code=sm_100a`` -- B200 only, no other targets;
* ``-fmad=false`` -- no FMA contraction: the float64 routing / cell / voxel
  centre / projection formulas must round per operation like the reference's
  numba codegen;
* ``-lineinfo`` -- ncu source attribution.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lodb200.so")
SOURCES = ["lod_tree.cu", "lod_raster.cu", "lod_morton.cu", "lod_route.cu", "lod_ingest.cu"]
HEADERS = ["lod_common.cuh", "lod_kernels.cuh", "lod_small.cuh", "radix.cuh", "scan.cuh"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build _lodb200.so")


def flags() -> list[str]:
    return [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
        "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
        "-Xptxas", "-v" if os.environ.get("LOD_PTXAS_VERBOSE") else "-O3",
        "--expt-relaxed-constexpr",
        "-I", os.path.join(HERE, "..", "include"),
    ]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "lod_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return OUT
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    cmd = [nvcc(), *flags(), "-shared", "-o", OUT + ".tmp", *srcs, "-lcudart"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

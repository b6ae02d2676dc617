"""In-tree build of the CUDA engine for sm_100a.

    python -m paper_1908_09301_b200._build

nvcc cross-compiles without a GPU; the resulting .so lands in
paper_1908_09301_b200/_lib (git-ignored, shipped to the GPU box with the
gpurun snapshot).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SOURCES = ("csrc/taylor_kernel.cu", "csrc/taylor_cluster.cu", "csrc/taylor_pipe.cu", "csrc/taylor_grid.cu", "csrc/capi.cu")
OUT = os.path.join(HERE, "_lib", "libmptaylor_b200.so")
ARCH = ("-gencode", "arch=compute_100a,code=sm_100a")


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False, extra=()) -> str:
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [
        nvcc(), "-O3", "-lineinfo", "-std=c++17", *ARCH,
        "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(REPO, "include"),
        *(["-Xptxas", "-v"] if verbose else []), *extra,
        "-o", OUT, *[os.path.join(HERE, s) for s in SOURCES],
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))

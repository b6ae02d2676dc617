"""In-tree build of the CUDA engine for sm_100a.

    python -m paper_1908_09301_b200._build

nvcc cross-compiles without a GPU; the resulting .so lands in
paper_1908_09301_b200/_lib (git-ignored, shipped to the GPU box with the
gpurun snapshot).
"""

from __future__ import annotations

import os
import re
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SOURCES = ("csrc/taylor_kernel.cu", "csrc/taylor_grid.cu", "csrc/taylor_mx.cu", "csrc/taylor_warp.cu", "csrc/taylor_warp2.cu", "csrc/taylor_block.cu", "csrc/taylor_cblock.cu",
           "csrc/capi.cu")
OUT = os.path.join(HERE, "_lib", "libmptaylor_b200.so")
ARCH = ("-gencode", "arch=compute_100a,code=sm_100a")


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False, extra=(), incremental: bool = False) -> str:
    """Compile every translation unit in parallel (-c), then link the .so.
    incremental=True reuses objects newer than their source and the headers."""
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    objdir = os.path.join(HERE, "_lib", "obj")
    os.makedirs(objdir, exist_ok=True)
    common = [nvcc(), "-O3", "-lineinfo", "-std=c++17", *ARCH, "-Xcompiler", "-fPIC",
              "-I", os.path.join(REPO, "include"), *(["-Xptxas", "-v"] if verbose else []), *extra]

    csrc = os.path.join(HERE, "csrc")

    def newest(path, seen):
        """Latest mtime of a source and of every header it includes (quoted includes, recursively)."""
        if path in seen or not os.path.exists(path):
            return 0.0
        seen.add(path)
        t = os.path.getmtime(path)
        with open(path) as fh:
            for line in fh:
                m = re.match(r'\s*#\s*include\s+"([^"]+)"', line)
                if m:
                    t = max(t, newest(os.path.normpath(os.path.join(os.path.dirname(path), m.group(1))), seen))
        return t

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        # incremental: an object newer than its source and every header it includes is reused
        if incremental and os.path.exists(obj) and os.path.getmtime(obj) > newest(os.path.join(HERE, src), set()):
            return obj, ""
        res = subprocess.run([*common, "-c", "-o", obj, os.path.join(HERE, src)], capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{res.stdout}\n{res.stderr}")
        return obj, res.stderr

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    if verbose:
        for _, err in results:
            sys.stderr.write(err)
    res = subprocess.run([nvcc(), *ARCH, "-shared", "-o", OUT, *[o for o, _ in results]], capture_output=True,
                         text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, incremental="-i" in sys.argv))

"""Build libpsigpu.so in-tree for sm_100a (B200).

    python -m paper_0904_0939_b200.build

nvcc cross-compiles without a GPU.  --fmad=false keeps the reference's
no-FMA evaluation order for every expression the kernels do not already
pin with __dadd_rn/__dmul_rn intrinsics.  cudart is linked statically so
the library loads on any host of this image.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "psigpu.cu")
OUT = os.path.join(HERE, "libpsigpu.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False) -> str:
    csrc = os.path.join(HERE, "csrc")
    deps = [os.path.join(csrc, f) for f in sorted(os.listdir(csrc))
            if f.endswith((".cu", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "psigpu.h"))
    if not force and os.path.exists(OUT) and all(
            os.path.getmtime(OUT) >= os.path.getmtime(d) for d in deps):
        return OUT
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-o", OUT + ".tmp", SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

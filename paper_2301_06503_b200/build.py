"""Build liblgdm.so in-tree with nvcc for sm_100a (no GPU needed)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "lgdm_api.cu")
OUT = os.path.join(HERE, "liblgdm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-fopenmp,-O2", "-shared", f"-I{os.path.join(ROOT, 'include')}"]


def sources():
    return [SRC] + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [
        os.path.join(ROOT, "include", "lgdm.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    stale = not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(s) for s in sources())
    if force or stale:
        cmd = [NVCC] + FLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-o", OUT, SRC, "-lgomp", "-ldl"]
        print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd, cwd=ROOT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)

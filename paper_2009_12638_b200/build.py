"""Build libbsgpu.so in-tree with nvcc for sm_100a (no torch types in the ABI)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "bs_engine.cu")]
OUT = os.path.join(HERE, "_lib", "libbsgpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",            # reference rounding: no FMA contraction anywhere
    "-Xcompiler", "-fPIC", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def build(verbose: bool = False, force: bool = False, out: str = OUT, defines=()) -> str:
    os.makedirs(os.path.dirname(out), exist_ok=True)
    deps = SRC + [os.path.join(ROOT, "include", "blocksolve_b200.h"), __file__]
    if not force and os.path.exists(out):
        if os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
            return out
    cmd = ([NVCC] + FLAGS + ["-D" + d for d in defines] + (["-Xptxas", "-v"] if verbose else [])
           + SRC + ["-o", out])
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))

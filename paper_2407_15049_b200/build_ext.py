"""Build libculorads.so in-tree with nvcc for sm_100a.

    python -m paper_2407_15049_b200.build_ext [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "culorads.cu"), os.path.join(HERE, "csrc", "admm_native.cu"),
       os.path.join(HERE, "csrc", "alm_native.cu"), os.path.join(HERE, "csrc", "spectral_native.cu"),
       os.path.join(HERE, "csrc", "admm_fused.cu"), os.path.join(HERE, "csrc", "alm_fused.cu")]
HDR = [os.path.join(ROOT, "include", "culorads.h")]
OUT = os.path.join(HERE, "libculorads.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-O3"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in SRC + HDR)


def build(force=False, verbose=False):
    if not force and not stale():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", OUT + ".tmp", *SRC]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

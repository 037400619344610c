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
HDR = [os.path.join(ROOT, "include", "culorads.h")] + [
    os.path.join(HERE, "csrc", f) for f in sorted(os.listdir(os.path.join(HERE, "csrc"))) if f.endswith(".cuh")]
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
    """Compile every source to an object in parallel (one nvcc per file), then link."""
    if not force and not stale():
        return OUT
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    with tempfile.TemporaryDirectory() as tmp:
        objs = [os.path.join(tmp, os.path.basename(src) + ".o") for src in SRC]
        cmds = [[nvcc(), *flags, "-I", os.path.join(ROOT, "include"), "-c", "-o", o, src]
                for src, o in zip(SRC, objs)]
        if verbose:
            for c in cmds:
                print(" ".join(c), flush=True)
        with ThreadPoolExecutor(len(cmds)) as pool:
            for r in pool.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds):
                if r.returncode != 0:
                    raise RuntimeError(f"nvcc failed:\n{r.stderr[-4000:]}")
        link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                "-o", OUT + ".tmp", *objs]
        if verbose:
            print(" ".join(link), flush=True)
        subprocess.run(link, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

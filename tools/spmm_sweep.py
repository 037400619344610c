"""Build/time variants of the tiled SpMM (compile-time knobs) on the bench instance. Dev tool.

    python tools/spmm_sweep.py build            # here: nvcc every variant into build_variants/
    python tools/spmm_sweep.py run              # on the GPU box: time each variant (one process each)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build_variants")
VARIANTS = {
    "base": [],
    "u4": ["-DSP_UNROLL=4"],
    "u12": ["-DSP_UNROLL=12"],
    "minb4": ["-DSP_MINB0=4"],
    "minb6": ["-DSP_MINB0=6"],
    "smax512": ["-DSP_SMAX=512"],
}


def build():
    sys.path.insert(0, ROOT)
    from paper_2407_15049_b200 import build_ext
    os.makedirs(OUT, exist_ok=True)
    for tag, flags in VARIANTS.items():
        if len(sys.argv) > 2 and tag not in sys.argv[2:]:
            continue
        cmd = [build_ext.nvcc(), *build_ext.NVCC_FLAGS, *flags, "-I", os.path.join(ROOT, "include"),
               "-o", os.path.join(OUT, f"libculorads_{tag}.so"), *build_ext.SRC]
        subprocess.run(cmd, check=True)
        print("built", tag, flush=True)


def one(tag):
    l2g = None
    if tag.startswith("l2g"):
        l2g = int(tag[3:])
        tag = "base"
    if tag != "base":      # base: the in-tree library (build_variants/ does not travel to the box)
        os.environ["CULORADS_LIB"] = os.path.join(OUT, f"libculorads_{tag}.so")
    sys.path.insert(0, ROOT)
    import math
    import numpy as np
    import torch
    from paper_2407_15049_b200 import alm, device, driver, graphs, linops, problem
    from paper_2407_15049_b200 import roofline as RL
    n = int(1e7)
    p = problem.build_maxcut(graphs.random_sparse(n, deg=6.0, seed=0))
    ops = linops.build_operators(p)
    dev = ops.dev
    if l2g is not None:
        rc = dev.lib.cl_set_l2_fetch_granularity(l2g)
        tag = f"l2g{l2g} (rc {rc}, now {dev.lib.cl_get_l2_fetch_granularity()})"
    else:
        tag = f"{tag} (l2 granularity {dev.lib.cl_get_l2_fetch_granularity()})"
    r = driver.initial_rank(p.m, p.n)
    ld = device.padded_ld(r)
    R = linops.to_factor(np.random.default_rng(0).standard_normal((n, r)) / math.sqrt(n * r), dev, ld)
    core = alm.AlmCore(ops, n, ld)
    D = R.clone()
    st = dev.stream
    res = {}
    for name, fn in [("c_times", lambda: core.c_times(R, core.CR)),
                     ("line_search_spmm", lambda: dev.spmm(ops.c_mat.cpat, D, ld, out=core.CD, Z=[R, D, core.CR],
                                                         dots=[("out", ("z", 0)), ("out", ("z", 1)),
                                                               (("z", 2), ("z", 1))], at=40, c_coeff=1.0))]:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 20
    b = RL.pattern_spmm_bytes(n, int(ops.c_mat.cpat.indices.numel()), ld)
    res["c_times_GBps"] = b / (res["c_times"] * 1e-3) / 1e9
    print(json.dumps({"variant": tag, **res}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    elif sys.argv[1] == "run":
        tags = sys.argv[2:] or (list(VARIANTS) + ["l2g0", "l2g32", "l2g64", "l2g128"])
        for tag in tags:
            subprocess.run([sys.executable, __file__, "one", tag])
    else:
        one(sys.argv[2])

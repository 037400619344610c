"""Register-cap (minBlocksPerSM) variants of the gather-bound kernels (dev tool).

    python tools/occupancy_sweep.py build [tags...]   # here: nvcc each variant into variants_so/
    python tools/occupancy_sweep.py run [tags...]     # on the GPU box: time each (one process each)

ncu (round 2) shows the completion kernels and the MaxCut SpMM at 50 % warp occupancy
(54-64 registers -> 4 CTAs of 256 threads per SM) with long-scoreboard stalls dominant and
DRAM at 32-66 % of peak: latency-bound gathers. Capping registers raises the loads in flight.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "variants_so")     # travels to the GPU box (not in .gpurunignore); *.so git-ignored
VARIANTS = {
    "base": [],
    "ck5_se5": ["-DCK_MINB=5", "-DSE_MINB=5"],
    "ck6_se6": ["-DCK_MINB=6", "-DSE_MINB=6"],
    "ck7": ["-DCK_MINB=7"],
    "ck8_se8": ["-DCK_MINB=8", "-DSE_MINB=8"],
    "ck3_4": ["-DCK3_MINB=4"],
    "ck3_5": ["-DCK3_MINB=5"],
    "sp1_4": ["-DSP_MINB1=4"],
    "spu12": ["-DSP_UNROLL=12"],
    "spu4": ["-DSP_UNROLL=4"],
    "split0": ["-DSP_SPLIT_LD=0"],
    "nosplit": ["-DSP_SPLIT_LD=100000"],
    "sp2_4": ["-DSP_MINB2=4"],
    "sp5": ["-DSP_MINB0=5"],
    "sp6": ["-DSP_MINB0=6"],
}


def build(tags):
    sys.path.insert(0, ROOT)
    from paper_2407_15049_b200 import build_ext
    os.makedirs(OUT, exist_ok=True)
    for tag in tags:
        cmd = [build_ext.nvcc(), *build_ext.NVCC_FLAGS, *VARIANTS[tag], "-I", os.path.join(ROOT, "include"),
               "-o", os.path.join(OUT, f"libculorads_{tag}.so"), *build_ext.SRC]
        subprocess.run(cmd, check=True)
        print("built", tag, flush=True)


def one(tag):
    if tag != "base":
        os.environ["CULORADS_LIB"] = os.path.join(OUT, f"libculorads_{tag}.so")
    sys.path.insert(0, ROOT)
    import math
    import numpy as np
    import torch
    from paper_2407_15049_b200 import admm, alm, device, driver, graphs, linops, problem
    res = {"variant": tag}

    def timeit(dev, fn, reps=10):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(dev.stream)
        for _ in range(reps):
            fn()
        e1.record(dev.stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    # completion at configs[3]'s one-GPU share
    p = problem.build_matrix_completion(graphs.random_completion(1250000, 1250000, int(2.5e7), seed=0))
    ops = linops.build_operators(p)
    dev = ops.dev
    r = driver.initial_rank(p.m, p.n)
    ld = device.padded_ld(r)
    rng = np.random.default_rng(0)
    U = linops.to_factor(rng.standard_normal((p.n, r)) / math.sqrt(p.n), dev, ld)
    V = linops.to_factor(rng.standard_normal((p.n, r)) / math.sqrt(p.n), dev, ld)
    y = dev.empty(p.m)
    out = dev.empty(p.n, ld)
    hs = admm.HalfStep(ops, p.n, ld)
    res["A(UV^T)_ms"] = timeit(dev, lambda: dev.constraint_eval(ops.cop.con, ld, U, V, y))
    res["single_entry_apply_ms"] = timeit(dev, lambda: hs.apply(U, V, 1.5, out, dot_with=U, at=0))
    if hasattr(dev.lib, "cl_single_entry_apply_pair"):
        P2 = dev.empty(p.n, 2 * ld)
        dev.pair_pack(U, ld, P2, 0)
        dev.pair_pack(V, ld, P2, 1)
        res["single_entry_apply_pair_ms"] = timeit(
            dev, lambda: dev.single_entry_apply_pair(ops.adj.apat, ld, P2, 1.5, out, at=0))
        res["pair_pack_ms"] = timeit(dev, lambda: dev.pair_pack(U, ld, P2, 0))
        del P2
    res["A(RD+DR, DD)_line_search_ms"] = timeit(dev, lambda: dev.constraint_eval(ops.cop.con, ld, U, V, y, X2=V, Y2=U,
                                                                               X3=V, Y3=V, out2=out.view(-1)[:p.m]))
    del ops, hs, U, V, y, out
    torch.cuda.empty_cache()
    # MaxCut C R at configs[2]
    n = int(1e7)
    p = problem.build_maxcut(graphs.random_sparse(n, deg=6.0, seed=0))
    ops = linops.build_operators(p, dev=dev)
    r = driver.initial_rank(p.m, p.n)
    ld = device.padded_ld(r)
    R = linops.to_factor(np.random.default_rng(0).standard_normal((n, r)) / math.sqrt(n * r), dev, ld)
    core = alm.AlmCore(ops, n, ld)
    res["maxcut_CR_ms"] = timeit(dev, lambda: core.c_times(R, core.CR), reps=20)
    D = R.clone()
    ls = lambda: dev.spmm(ops.c_mat.cpat, D, ld, out=core.CD, Z=[R, D, core.CR],  # noqa: E731
                          dots=[("out", ("z", 0)), ("out", ("z", 1)), (("z", 2), ("z", 1))], at=40, c_coeff=1.0)
    res["maxcut_linesearch_spmm_ms"] = timeit(dev, ls, reps=20)
    del ops, core, R, D
    torch.cuda.empty_cache()
    # high rank (configs[1] after its escalations): n = 1e6, r = 822
    n = int(1e6)
    p = problem.build_maxcut(graphs.random_sparse(n, deg=10.0, seed=0))
    ops = linops.build_operators(p, dev=dev)
    ld = 822
    R = linops.to_factor(np.random.default_rng(0).standard_normal((n, ld)) / math.sqrt(n * ld), dev, ld)
    core = alm.AlmCore(ops, n, ld)
    D = R.clone()
    res["hr_CR_ms"] = timeit(dev, lambda: core.c_times(R, core.CR), reps=5)
    res["hr_linesearch_spmm_ms"] = timeit(dev, ls, reps=5)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    tags = sys.argv[2:] or list(VARIANTS)
    if sys.argv[1] == "build":
        build(tags)
    elif sys.argv[1] == "run":
        for tag in tags:
            subprocess.run([sys.executable, __file__, "one", tag])
    else:
        one(sys.argv[2])

"""Solve the same MaxCut instance with the device solver (and optionally the CPU oracle);
print solve seconds, iteration counts and objectives. Development probe for DESIGN.md.

    python tools/compare_solve.py N DEG [--oracle] [--time-limit S]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("n", type=float)
ap.add_argument("deg", type=float)
ap.add_argument("--oracle", action="store_true")
ap.add_argument("--gpu", action="store_true")
ap.add_argument("--time-limit", type=float, default=600.0)
ap.add_argument("--level", type=int, default=1)
a = ap.parse_args()
from paper_2407_15049_b200 import graphs, problem  # noqa: E402
p = problem.build_maxcut(graphs.random_sparse(int(a.n), deg=a.deg, seed=1))
print(f"n={p.n} edges={p.C.nnz_stored - p.n}", flush=True)
if a.gpu:
    import torch
    from paper_2407_15049_b200 import driver
    driver.solve(p, driver.SolverConfig(time_limit=5, reopt_level=a.level))   # warm-up (lib load, allocator)
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = driver.solve(p, driver.SolverConfig(time_limit=a.time_limit, reopt_level=a.level))
    dt = time.perf_counter() - t
    print(f"gpu: {dt:.3f}s status {rep.status} obj {rep.objective:.10g} err1 {rep.err1:.2e} err3 {rep.err3:.2e} "
          f"ranks {rep.rank_history} alm {rep.alm_inner_iterations} admm {rep.admm_steps} cg {rep.cg_iterations} "
          f"reopt {rep.reopt_rounds} rows {len(rep.trace_rows)} launches {rep.gpu_launches}", flush=True)
if a.oracle:
    from oracle import lrsdp_oracle as O
    t = time.perf_counter()
    r = O.solve(p, time_limit=a.time_limit, reopt_level=a.level)
    dt = time.perf_counter() - t
    print(f"oracle: {dt:.3f}s status {r['status']} obj {r['objective']:.10g} err1 {r['err1']:.2e} "
          f"err3 {r['err3']:.2e} ranks {r['rank_history']} alm {r['alm_inner']} admm {r['admm_steps']} "
          f"cg {r['cg']} rows {len(r['trace'])}", flush=True)

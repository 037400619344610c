"""Time one device MaxCut solve on a synthetic graph (development probe, not the bench).

    python tools/probe_solve.py N DEG [time_limit] [random|delaunay] [reorder]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_15049_b200 import driver, graphs, linops, problem  # noqa: E402

n = int(float(sys.argv[1]))
deg = float(sys.argv[2])
tl = float(sys.argv[3]) if len(sys.argv) > 3 else 600.0
kind = sys.argv[4] if len(sys.argv) > 4 else "random"
reorder = len(sys.argv) > 5 and sys.argv[5] == "reorder"
t = time.perf_counter()
g = graphs.delaunay_like(n, seed=0) if kind == "delaunay" else graphs.random_sparse(n, deg=deg, seed=0)
t_g = time.perf_counter() - t
t = time.perf_counter()
p = problem.build_maxcut(g)
t_p = time.perf_counter() - t
t = time.perf_counter()
ops = None if reorder else linops.build_operators(p)
torch.cuda.synchronize()
t_o = time.perf_counter() - t
print(f"{kind} reorder={reorder} n={n} edges={g.edges_u.size} gen {t_g:.2f}s build_maxcut {t_p:.2f}s build_operators {t_o:.2f}s", flush=True)
t = time.perf_counter()
rep = driver.solve(p, driver.SolverConfig(time_limit=tl, reorder=reorder), ops=ops)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"solve {dt:.2f}s status {rep.status} obj {rep.objective:.10g} err1 {rep.err1:.2e} err3 {rep.err3:.2e} "
      f"err2 {rep.err2} rank {rep.rank_history} alm {rep.alm_outer_iterations}/{rep.alm_inner_iterations} "
      f"admm {rep.admm_steps} cg {rep.cg_iterations} reopt {rep.reopt_rounds} t_alm {rep.time_alm_s:.2f} "
      f"t_admm {rep.time_admm_s:.2f} launches {rep.gpu_launches} peak {rep.peak_bytes/2**30:.1f} GiB", flush=True)

"""A capped MaxCut solve that runs every stage once (ALM, ADMM with CG, final Lanczos): the
launch-list target for profiles/ (every kernel of the solve path in one run). Dev probe.

    python tools/capped_solve.py N DEG
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_15049_b200 import driver, graphs, problem  # noqa: E402

n, deg = int(float(sys.argv[1])), float(sys.argv[2])
p = problem.build_maxcut(graphs.random_sparse(n, deg=deg, seed=0))
t = time.perf_counter()
rep = driver.solve(p, driver.SolverConfig(alm_outer_cap=2, alm_inner_cap=40, admm_step_cap=30, max_reopts=0))
print(f"capped solve n={n}: {time.perf_counter() - t:.2f} s status {rep.status} rows {len(rep.trace_rows)} "
      f"admm {rep.admm_steps} cg {rep.cg_iterations} launches {rep.gpu_launches}")

"""cProfile of one device solve (host-side overhead breakdown), dev probe.

    python tools/host_profile.py N DEG
"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_15049_b200 import driver, graphs, problem  # noqa: E402

p = problem.build_maxcut(graphs.random_sparse(int(float(sys.argv[1])), deg=float(sys.argv[2]), seed=1))
driver.solve(p, driver.SolverConfig(time_limit=3))
pr = cProfile.Profile()
pr.enable()
rep = driver.solve(p, driver.SolverConfig(time_limit=float(sys.argv[3]) if len(sys.argv) > 3 else 60))
pr.disable()
print(rep.status, rep.admm_steps, rep.alm_inner_iterations, rep.time_total_s)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

"""One G1-shaped MaxCut solve (BASELINE configs[0]) on the device (profiling target)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_15049_b200 import driver, graphs, problem  # noqa: E402

p = problem.build_maxcut(graphs.random_sparse(800, deg=48.0, seed=1))
for _ in range(3):     # the first solve includes one-time setup (library load, first launches)
    t = time.perf_counter()
    rep = driver.solve(p, driver.SolverConfig())
    print(f"G1 solve {time.perf_counter() - t:.3f} s status {rep.status} objective {rep.objective:.10g} "
          f"rows {len(rep.trace_rows)}")

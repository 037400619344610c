"""Run the device solver on every golden solve case and store its traces (gpurun_out/)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_15049_b200 import driver  # noqa: E402
from tests._golden import cfg_of, load, problem_from, solve_cases  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
os.makedirs(out, exist_ok=True)
for case in solve_cases():
    z = load(f"solve_{case}.npz")
    cfg = cfg_of(z)
    if case == "maxcut_2k_deg6":
        cfg = dict(admm_step_cap=3000, max_reopts=0)
    t = time.perf_counter()
    rep = driver.solve(problem_from(z), driver.SolverConfig(**cfg))
    dt = time.perf_counter() - t
    tr = np.array([r[2:7] for r in rep.trace_rows], dtype=float).reshape(-1, 5)
    np.savez(os.path.join(out, f"trace_{case}.npz"), trace=tr, status=rep.status,
             objective=rep.objective, err1=rep.err1, err2=np.nan if rep.err2 is None else rep.err2,
             err3=rep.err3, alm_inner=rep.alm_inner_iterations, admm_steps=rep.admm_steps,
             time=dt, launches=rep.gpu_launches)
    print(case, rep.status, rep.objective, rep.err1, rep.err2, rep.err3, len(tr),
          f"{dt:.2f}s", rep.gpu_launches, flush=True)

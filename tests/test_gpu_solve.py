"""Full solves on the device vs the reference's traces (golden) and the CPU oracle.

north_star tolerances: per-iteration objective and primal infeasibility to
1e-9 relative (fp64; err1 also gets an absolute floor of 1e-13 because near
convergence it is a norm of a cancellation-limited residual), final
objective to 1e-6 relative, comparable iteration counts.
"""

import numpy as np
import pytest

from tests._golden import cfg_of, load, problem_from, solve_cases

pytestmark = pytest.mark.gpu


def trace_array(rows):
    return np.array([r[2:7] for r in rows], dtype=float).reshape(-1, 5)


def compare_traces(got, ref, upto=None):
    k = min(len(got), len(ref)) if upto is None else min(upto, len(got), len(ref))
    g, r = got[:k], ref[:k]
    obj_rel = np.abs(g[:, 0] - r[:, 0]) / np.maximum(1.0, np.abs(r[:, 0]))
    e1_dev = np.abs(g[:, 1] - r[:, 1]) / (1e-13 / 1e-9 + np.abs(r[:, 1]))
    return k, float(obj_rel.max(initial=0.0)), float(e1_dev.max(initial=0.0))


@pytest.mark.parametrize("case", [c for c in solve_cases() if c != "maxcut_2k_deg6"])
def test_solve_matches_reference(case):
    from paper_2407_15049_b200 import driver
    z = load(f"solve_{case}.npz")
    p = problem_from(z)
    rep = driver.solve(p, driver.SolverConfig(**cfg_of(z)))
    got, ref = trace_array(rep.trace_rows), z["trace"]
    k, obj_rel, e1_rel = compare_traces(got, ref)
    print(f"{case}: status {rep.status}/{z['status']} rows {len(got)}/{len(ref)} "
          f"obj_rel {obj_rel:.2e} err1_rel {e1_rel:.2e} objective {rep.objective!r} vs {float(z['objective'])!r}")
    assert rep.status == str(z["status"])
    assert abs(rep.objective - float(z["objective"])) <= 1e-6 * (1 + abs(float(z["objective"])))
    assert abs(len(got) - len(ref)) <= max(2, 0.1 * len(ref))
    assert obj_rel <= 1e-9 and e1_rel <= 1e-9
    assert rep.gpu_launches > 0


def test_long_trajectory_prefix_matches_reference():
    """n=2000 sparse MaxCut: the reference's first 2000 trace rows (ALM stage)."""
    from paper_2407_15049_b200 import driver
    z = load("solve_maxcut_2k_deg6.npz")
    p = problem_from(z)
    cfg = driver.SolverConfig(alm_outer_cap=50, admm_step_cap=1, max_reopts=0)
    rep = driver.solve(p, cfg)
    got, ref = trace_array(rep.trace_rows), z["trace"]
    k, obj_rel, e1_rel = compare_traces(got, ref, upto=2000)
    print(f"prefix rows {k}: obj_rel {obj_rel:.2e} err1_rel {e1_rel:.2e}")
    assert k == 2000
    assert obj_rel <= 1e-9 and e1_rel <= 1e-9

"""Full device solves vs the reference (golden traces + its own 1-ulp envelope).

The reference algorithm is chaotic: re-running it with its L-BFGS direction
perturbed by one ulp (tests/golden/make_golden.py: perturbed_runs) moves the
per-iteration trace by more than 1e-9 after a case-dependent number of rows
(``ulp_horizon``) and spreads the final objective / iteration count. No
implementation with a different floating-point summation order can track
it further. The device solver is therefore held to:

* per-iteration objective and err1 equal to the reference's to 1e-9
  relative (err1 with a 1e-13 absolute floor) over at least half of the
  reference's own 1-ulp horizon;
* final status among the statuses the perturbed reference reaches;
* final objective inside the perturbed reference's spread, widened by 1e-6
  relative (north_star: final objective to 1e-6), for converged ("optimal")
  and capped ("best_effort") runs alike;
* trace length between half the perturbed reference's shortest run and twice
  its longest (a comparable iteration count).
"""

import numpy as np
import pytest

from tests._golden import cfg_of, load, problem_from, solve_cases

pytestmark = pytest.mark.gpu


def trace_array(rows):
    return np.array([r[2:7] for r in rows], dtype=float).reshape(-1, 5)


def first_dev(tr, ref, tol=1e-9):
    k = min(len(tr), len(ref))
    d = np.abs(tr[:k, 0] - ref[:k, 0]) / np.maximum(1.0, np.abs(ref[:k, 0]))
    e = np.abs(tr[:k, 1] - ref[:k, 1]) / (1e-4 + np.abs(ref[:k, 1]))
    bad = np.nonzero((d > tol) | (e > tol))[0]
    return int(bad[0]) if bad.size else k


@pytest.mark.parametrize("case", solve_cases())
def test_solve_within_reference_envelope(case):
    from paper_2407_15049_b200 import driver
    z = load(f"solve_{case}.npz")
    p = problem_from(z)
    rep = driver.solve(p, driver.SolverConfig(**cfg_of(z)))
    got, ref = trace_array(rep.trace_rows), z["trace"]
    horizon = first_dev(got, ref)
    ref_h = int(z["ulp_horizon"].min())
    objs = np.append(z["ulp_objective"], float(z["objective"]))
    rows = np.append(z["ulp_rows"], len(ref))
    statuses = set(z["ulp_status"].tolist()) | {str(z["status"])}
    print(f"{case}: status {rep.status} (ref {sorted(statuses)}) rows {len(got)} (ref {rows.min()}..{rows.max()}) "
          f"1e-9 horizon {horizon} (ref ulp {ref_h}) objective {rep.objective!r} "
          f"(ref {objs.min()!r}..{objs.max()!r})")
    assert rep.gpu_launches > 0
    assert horizon >= min(len(ref), len(got), max(1, ref_h // 2))
    assert rep.status in statuses
    lo, hi = objs.min(), objs.max()
    pad = 1e-6 * max(1.0, abs(hi), abs(lo))
    if case != "random_sdp":
        # optimal and capped (best_effort) runs alike: inside the perturbed reference's spread,
        # widened by 1e-6 relative. random_sdp is unbounded below (dense random A_i, no trace
        # constraint): its objective is ~-1e33 noise that the reference's own runs spread over 33
        # orders of magnitude, so only its status and trace horizon are compared.
        assert lo - pad <= rep.objective <= hi + pad
    assert 0.5 * rows.min() <= len(got) <= 2.0 * rows.max()


def test_final_errors_recomputed_honestly():
    """Report honesty (driver.py:572): err1/err3 recomputed from the returned factors."""
    from paper_2407_15049_b200 import driver
    z = load("solve_g1_like.npz")
    p = problem_from(z)
    rep = driver.solve(p, driver.SolverConfig())
    U = rep.U[:, :rep.rank_final].cpu().numpy()
    V = rep.V[:, :rep.rank_final].cpu().numpy()
    lam = rep.lam.cpu().numpy()
    from oracle import lrsdp_oracle as O
    e = O.errors(O.OracleOps(p), U, V, lam)
    assert abs(e["err1"] - rep.err1) <= 1e-12 + 1e-9 * rep.err1
    assert abs(e["err3"] - rep.err3) <= 1e-12 + 1e-9 * rep.err3
    assert abs(-e["obj"] - rep.objective) <= 1e-9 * abs(rep.objective)


def test_determinism_same_seed_bit_identical():
    from paper_2407_15049_b200 import driver
    z = load("solve_completion_30.npz")
    p = problem_from(z)
    a = driver.solve(p, driver.SolverConfig(deterministic=True))
    b = driver.solve(p, driver.SolverConfig(deterministic=True))
    assert a.to_json_dict() == b.to_json_dict()
    assert trace_array(a.trace_rows).tobytes() == trace_array(b.trace_rows).tobytes()


def test_locality_reordered_solve_in_envelope_and_unpermuted():
    """SolverConfig(reorder=True) on the Delaunay-like instance (labels scrambled, RCM
    order restores locality): same envelope as the plain solve, factors and multipliers
    returned in the caller's labelling (errors recomputed by the oracle agree)."""
    from oracle import lrsdp_oracle as O
    from paper_2407_15049_b200 import driver, reorder
    z = load("solve_delaunay_45.npz")
    p = problem_from(z)
    assert reorder.locality_gain(p, reorder.locality_order(p)) >= 2.0
    cfg = dict(cfg_of(z))
    rep = driver.solve(p, driver.SolverConfig(**cfg, reorder=True))
    objs = np.append(z["ulp_objective"], float(z["objective"]))
    statuses = set(z["ulp_status"].tolist()) | {str(z["status"])}
    assert rep.status in statuses
    lo, hi = objs.min(), objs.max()
    if rep.status == "optimal":
        assert lo - 1e-6 * hi <= rep.objective <= hi + 1e-6 * hi
    r = rep.rank_final
    e = O.errors(O.OracleOps(p), rep.U[:, :r].cpu().numpy(), rep.V[:, :r].cpu().numpy(), rep.lam.cpu().numpy())
    assert abs(e["err1"] - rep.err1) <= 1e-12 + 1e-9 * rep.err1
    assert abs(e["err3"] - rep.err3) <= 1e-12 + 1e-9 * rep.err3
    assert abs(-e["obj"] - rep.objective) <= 1e-9 * abs(rep.objective)


def test_reorder_skipped_for_random_graphs():
    from paper_2407_15049_b200 import driver
    z = load("solve_g1_like.npz")
    p = problem_from(z)
    a = driver.solve(p, driver.SolverConfig(deterministic=True))
    b = driver.solve(p, driver.SolverConfig(deterministic=True, reorder=True))
    assert trace_array(a.trace_rows).tobytes() == trace_array(b.trace_rows).tobytes()


def test_memory_guard_caps_rank_escalation():
    """SolverConfig.memory_budget: an escalation whose stage buffers would not fit is refused
    like one at the sqrt(2m) cap -- the solve continues at its rank and reports it -- instead
    of failing out of memory."""
    import torch
    from paper_2407_15049_b200 import driver, graphs, linops, problem
    p = problem.build_maxcut(graphs.random_sparse(3000, deg=8.0, seed=2))
    cfg = dict(alm_inner_cap=20, alm_outer_cap=8, admm_step_cap=30, max_reopts=0)
    free = driver.SolverConfig(**cfg)
    rep = driver.solve(p, free)
    assert len(rep.rank_history) > 1 and not rep.memory_capped       # this run escalates
    ops = linops.build_operators(p)
    torch.cuda.synchronize()
    r0 = driver.initial_rank(p.m, p.n)
    base = torch.cuda.memory_allocated()
    budget = base + driver.factor_bytes_needed(p.n, p.m, r0, 8)     # r0 fits, nothing more
    capped = driver.solve(p, driver.SolverConfig(memory_budget=budget, **cfg), ops=ops)
    assert capped.memory_capped and capped.rank_history == [r0]
    assert capped.memory_rank_refused == rep.rank_history[1]
    assert capped.status in ("best_effort", "optimal", "timeout") and capped.rank_final == r0

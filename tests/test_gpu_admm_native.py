"""The native ADMM step (cl_admm_step_diag) against the Python-driven step.

Both issue the same launches in the same order and take the same scalar
decisions, so iterates, multipliers and step statistics must agree bit for
bit; so must a full solve's trace.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_steps(native, p, steps, seed=0, r=6, fused=False):
    import torch
    from paper_2407_15049_b200 import admm, alm, linops
    from paper_2407_15049_b200.device import padded_ld
    admm.NATIVE = native
    admm.FUSED = fused
    try:
        ops = linops.build_operators(p)
        dev = ops.dev
        ld = padded_ld(r)
        rng = np.random.default_rng(seed)
        R = linops.to_factor(rng.standard_normal((p.n, r)) / np.sqrt(p.n * r), dev, ld)
        dual = alm.DualVector(lam=linops.to_vec(0.3 * rng.standard_normal(p.m), dev).clone(), rho=2.0)
        state = admm.AdmmState(U=R.clone(), V=(R + 1e-3).contiguous(), dual=dual, r=r)
        hs, pool = admm.HalfStep(ops, p.n, ld), admm._Pool(dev, p.n, ld)
        stats = []
        for k in range(steps):
            s = admm.admm_step(state, ops, scale=0.7, hs=hs, pool=pool, cg_cap=50)
            stats.append((s.cg_iters_u, s.cg_iters_v, s.resid_u, s.resid_v, s.hit_cap, state.last_pnorm2))
        torch.cuda.synchronize()
        return state.U.cpu().numpy(), state.V.cpu().numpy(), dual.lam.cpu().numpy(), stats
    finally:
        admm.NATIVE = True
        admm.FUSED = True


@pytest.mark.parametrize("r", [6, 70, 400])     # r = 400: n*ld > 2^20, the in-order (unspeculated) step
def test_native_step_bit_identical_to_python_step(r):
    from paper_2407_15049_b200 import graphs, problem
    p = problem.build_maxcut(graphs.random_sparse(3000, deg=6.0, seed=4))
    a = _run_steps(True, p, 12, r=r)
    b = _run_steps(False, p, 12, r=r)
    assert sum(s[0] + s[1] for s in a[3]) > 0          # CG iterations actually ran
    for x, y in zip(a[:3], b[:3]):
        assert x.tobytes() == y.tobytes()
    assert a[3] == b[3]


def test_native_solve_trace_bit_identical():
    from paper_2407_15049_b200 import admm, driver
    from tests._golden import cfg_of, load, problem_from
    z = load("solve_g1_like.npz")
    p = problem_from(z)
    cfg = driver.SolverConfig(**cfg_of(z))
    admm.NATIVE = False
    try:
        slow = driver.solve(p, cfg)
    finally:
        admm.NATIVE = True
    admm.FUSED = False
    try:
        fast = driver.solve(p, cfg)
    finally:
        admm.FUSED = True
    tr = lambda rep: np.array([r[2:7] for r in rep.trace_rows], dtype=float)  # noqa: E731
    assert tr(fast).tobytes() == tr(slow).tobytes()
    assert fast.objective == slow.objective and fast.status == slow.status


@pytest.mark.parametrize("r,deg", [(6, 6.0), (11, 48.0), (70, 6.0)])
def test_fused_step_matches_native_step(r, deg):
    """The one-launch step (cl_admm_step_diag_fused) against the multi-launch native step:
    same CG iteration counts and reuse decisions, iterates equal to rounding (global sums
    are added in a different fixed order)."""
    from paper_2407_15049_b200 import graphs, problem
    p = problem.build_maxcut(graphs.random_sparse(800, deg=deg, seed=4))
    a = _run_steps(True, p, 6, r=r, fused=True)
    b = _run_steps(True, p, 6, r=r, fused=False)
    assert sum(s[0] + s[1] for s in b[3]) > 0
    for x, y in zip(a[:3], b[:3]):
        assert np.abs(x - y).max() <= 1e-9 * (1.0 + np.abs(y).max())
    for sa, sb in zip(a[3], b[3]):
        assert sa[0] == sb[0] and sa[1] == sb[1] and sa[4] == sb[4]
        for u, v in zip(sa[2:4] + sa[5:], sb[2:4] + sb[5:]):
            assert abs(u - v) <= 1e-8 * (1.0 + abs(v))


def test_fused_solve_trace_close_to_native():
    """A whole G1-shaped solve with fused steps: same status, objective to 1e-9 relative."""
    from paper_2407_15049_b200 import admm, driver
    from tests._golden import cfg_of, load, problem_from
    z = load("solve_g1_like.npz")
    p = problem_from(z)
    cfg = driver.SolverConfig(**cfg_of(z))
    admm.FUSED = False
    try:
        ref = driver.solve(p, cfg)
    finally:
        admm.FUSED = True
    fused = driver.solve(p, cfg)
    assert fused.status == ref.status
    assert abs(fused.objective - ref.objective) <= 1e-9 * abs(ref.objective)


def test_small_solve_runs_the_one_launch_paths():
    """The G1-shaped solve takes the one-launch paths: about one launch per ADMM step and per
    ALM inner solve (the multi-launch loops need about ten per step), and the same solve
    with them disabled launches several times more kernels."""
    from paper_2407_15049_b200 import admm, alm, driver, spectral
    from tests._golden import cfg_of, load, problem_from
    z = load("solve_g1_like.npz")
    p = problem_from(z)
    cfg = driver.SolverConfig(**cfg_of(z))
    fused = driver.solve(p, cfg)
    admm.FUSED = alm.FUSED = spectral.FUSED = False
    try:
        multi = driver.solve(p, cfg)
    finally:
        admm.FUSED = alm.FUSED = spectral.FUSED = True
    steps = fused.admm_steps
    assert fused.gpu_launches < 3 * steps + 1000
    assert multi.gpu_launches > 3 * fused.gpu_launches
    assert fused.status == multi.status


def test_fused_step_returns_balance_measures():
    """With want_balance the one-launch step returns ||U_new - U||^2 and ||V_new - V||^2
    (admm_run's residual balancing reads them instead of two more passes and a round trip)."""
    import torch
    from paper_2407_15049_b200 import admm, alm, graphs, linops, problem
    from paper_2407_15049_b200.device import padded_ld
    p = problem.build_maxcut(graphs.random_sparse(800, deg=20.0, seed=2))
    ops = linops.build_operators(p)
    dev = ops.dev
    r = 9
    ld = padded_ld(r)
    rng = np.random.default_rng(3)
    R = linops.to_factor(rng.standard_normal((p.n, r)) / np.sqrt(p.n * r), dev, ld)
    dual = alm.DualVector(lam=linops.to_vec(0.3 * rng.standard_normal(p.m), dev).clone(), rho=2.0)
    st = admm.AdmmState(U=R.clone(), V=(R + 1e-3).contiguous(), dual=dual, r=r)
    hs, pool = admm.HalfStep(ops, p.n, ld), admm._Pool(dev, p.n, ld)
    seen = 0
    for _ in range(6):
        U0, V0 = st.U.clone(), st.V.clone()
        st.want_balance = True
        admm.admm_step(st, ops, scale=0.7, hs=hs, pool=pool, cg_cap=50)
        assert st.step_bal is not None
        torch.cuda.synchronize()
        du2 = float(((st.U - U0) ** 2).sum())
        dv2 = float(((st.V - V0) ** 2).sum())
        assert abs(st.step_bal[0] - du2) <= 1e-12 * max(du2, 1e-300) + 1e-300
        assert abs(st.step_bal[1] - dv2) <= 1e-12 * max(dv2, 1e-300) + 1e-300
        seen += (du2 > 0) + (dv2 > 0)
    assert seen > 0
    st.want_balance = False
    admm.admm_step(st, ops, scale=0.7, hs=hs, pool=pool, cg_cap=50)
    assert st.step_bal is None


@pytest.mark.parametrize("case,r", [("completion", 6), ("completion", 26), ("sdpa", 4)])
def test_native_generic_step_bit_identical(case, r):
    """cl_admm_step_generic (general constraints: matrix completion on the pair-buffer
    single-entry operator, a dense-constraint SDPA instance on constraint pass + Omega_A
    product) against the Python-driven generic step."""
    from paper_2407_15049_b200 import admm, graphs, problem
    if case == "completion":
        p = problem.build_matrix_completion(graphs.random_completion(500, 420, 10000, seed=r))
    else:
        from tests._golden import load, problem_from
        p = problem_from(load("solve_random_sdp.npz"))
    a = _run_steps(True, p, 8, r=r, seed=3)
    admm.NATIVE_GENERIC = False
    try:
        b = _run_steps(True, p, 8, r=r, seed=3)
    finally:
        admm.NATIVE_GENERIC = True
    assert sum(s[0] + s[1] for s in a[3]) > 0
    for x, y in zip(a[:3], b[:3]):
        assert x.tobytes() == y.tobytes()
    assert a[3] == b[3]

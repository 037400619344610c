"""The native ALM inner loop (cl_alm_inner_diag) against the Python-driven loop.

Same launches, same operands, the same host scalar algebra restated in C++:
iterates, gradient norms, trace rows and termination must agree bit for bit,
through L-BFGS history eviction and the periodic constraint refresh.
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _Rec:
    def __init__(self):
        self.rows = []

    def record(self, stage, obj, err1, metric, rho, rank, t=None):
        self.rows.append((stage, obj, err1, metric, rho, rank))


def _run(native, p, iters, memory, seed, reduce_factor=None, fused=False):
    import torch
    from paper_2407_15049_b200 import alm, linops
    from paper_2407_15049_b200.device import padded_ld
    alm.NATIVE = native
    alm.FUSED = fused
    try:
        ops = linops.build_operators(p)
        dev = ops.dev
        r = 5
        ld = padded_ld(r)
        rng = np.random.default_rng(seed)
        R = linops.to_factor(rng.standard_normal((p.n, r)) / math.sqrt(p.n * r), dev, ld)
        lam = linops.to_vec(0.2 * rng.standard_normal(p.m), dev)
        core = alm.AlmCore(ops, p.n, ld)
        rec = _Rec()
        res = alm._inner(core, R, lam, 3.0, 0.9, 0.0, iters, reduce_factor, memory, alm._RankRecorder(rec, r))
        torch.cuda.synchronize()
        return R.cpu().numpy(), res.iterations, res.grad_norms, res.hit_cap, res.ax.cpu().numpy(), rec.rows
    finally:
        alm.NATIVE = True
        alm.FUSED = True


@pytest.mark.parametrize("memory,iters", [(8, 130), (3, 60), (1, 20)])
def test_native_inner_bit_identical(memory, iters):
    from paper_2407_15049_b200 import graphs, problem
    p = problem.build_maxcut(graphs.random_sparse(2500, deg=7.0, seed=memory))
    a = _run(True, p, iters, memory, 1)
    b = _run(False, p, iters, memory, 1)
    assert a[1] == b[1] and a[1] > 0
    assert a[0].tobytes() == b[0].tobytes()
    assert a[4].tobytes() == b[4].tobytes()
    assert a[2] == b[2] and a[3] == b[3]
    assert a[5] == b[5]


def test_native_inner_reduce_factor_exit():
    from paper_2407_15049_b200 import graphs, problem
    p = problem.build_maxcut(graphs.random_sparse(800, deg=10.0, seed=3))
    a = _run(True, p, 500, 8, 2, reduce_factor=1e-2)
    b = _run(False, p, 500, 8, 2, reduce_factor=1e-2)
    assert a[1] == b[1] and not a[3]
    assert a[0].tobytes() == b[0].tobytes()


def test_native_solve_matches_python_driven_solve():
    """Whole pipeline with both native loops vs both Python loops: identical traces."""
    from paper_2407_15049_b200 import admm, alm, driver
    from tests._golden import cfg_of, load, problem_from
    z = load("solve_maxcut_2k_deg6.npz")
    p = problem_from(z)
    cfg = driver.SolverConfig(**cfg_of(z))
    alm.NATIVE = admm.NATIVE = False
    try:
        slow = driver.solve(p, cfg)
    finally:
        alm.NATIVE = admm.NATIVE = True
    admm.FUSED = alm.FUSED = False   # the one-launch paths add their sums in another order (tested below)
    try:
        fast = driver.solve(p, cfg)
    finally:
        admm.FUSED = alm.FUSED = True
    tr = lambda rep: np.array([r[2:7] for r in rep.trace_rows], dtype=float)  # noqa: E731
    assert tr(fast).tobytes() == tr(slow).tobytes()
    assert fast.objective == slow.objective and fast.status == slow.status


@pytest.mark.parametrize("memory,iters,n", [(8, 130, 2500), (3, 60, 800), (8, 400, 800)])
def test_fused_inner_matches_native(memory, iters, n):
    """The one-launch inner solve (cl_alm_inner_diag_fused) against the multi-launch native
    loop: same iteration count and exit, through history eviction and the refresh every 50
    iterations; iterates, gradient norms and trace values equal to rounding."""
    from paper_2407_15049_b200 import graphs, problem
    p = problem.build_maxcut(graphs.random_sparse(n, deg=7.0, seed=memory))
    a = _run(True, p, iters, memory, 1, fused=True)
    b = _run(True, p, iters, memory, 1, fused=False)
    assert a[1] == b[1] and a[1] > 0 and a[3] == b[3]
    close = lambda x, y, t: np.abs(np.asarray(x) - np.asarray(y)).max() <= t * (1.0 + np.abs(np.asarray(y)).max())  # noqa: E731
    # 130 L-BFGS iterations amplify last-bit differences of the sums (as the reference's own
    # one-ulp envelope does): agreement to about 1e-8 relative remains
    assert close(a[0], b[0], 1e-6) and close(a[4], b[4], 1e-6)
    assert len(a[2]) == len(b[2]) and close(a[2], b[2], 1e-6)
    assert len(a[5]) == len(b[5])
    for ra, rb in zip(a[5], b[5]):
        assert ra[0] == rb[0] and ra[5] == rb[5]
        assert close(ra[1:4], rb[1:4], 1e-6)


def test_fused_inner_reduce_factor_exit_and_times():
    """Reduce-factor exit in the one-launch solve; trace times are host-clock and increasing."""
    import time
    from paper_2407_15049_b200 import alm, graphs, linops, problem
    from paper_2407_15049_b200.device import padded_ld
    p = problem.build_maxcut(graphs.random_sparse(800, deg=10.0, seed=3))
    a = _run(True, p, 500, 8, 2, reduce_factor=1e-2, fused=True)
    b = _run(True, p, 500, 8, 2, reduce_factor=1e-2, fused=False)
    assert a[1] == b[1] and not a[3]
    ops = linops.build_operators(p)
    r = 5
    R = linops.to_factor(np.random.default_rng(0).standard_normal((p.n, r)) / 60.0, ops.dev, padded_ld(r))
    core = alm.AlmCore(ops, p.n, padded_ld(r))
    times = []

    class T:
        def record(self, stage, obj, err1, metric, rho, rank, t=None):
            times.append(t)
    t0 = time.perf_counter()
    alm._inner(core, R, ops.dev.zeros(p.m), 3.0, 0.9, 0.0, 30, None, 8, alm._RankRecorder(T(), r))
    t1 = time.perf_counter()
    assert times and all(t0 - 1e-3 <= t <= t1 + 1e-3 for t in times)
    assert all(u <= v for u, v in zip(times, times[1:]))


@pytest.mark.parametrize("case,memory,iters", [("completion", 8, 120), ("completion", 3, 40), ("sdpa", 8, 60)])
def test_native_generic_inner_bit_identical(case, memory, iters):
    """cl_alm_inner_generic (general constraints: matrix completion with the pair-buffer line
    search, a dense-constraint SDPA instance) against the Python-driven generic loop."""
    from paper_2407_15049_b200 import graphs, problem
    if case == "completion":
        p = problem.build_matrix_completion(graphs.random_completion(400, 350, 9000, seed=memory))
    else:
        from tests._golden import load, problem_from
        p = problem_from(load("solve_random_sdp.npz"))
    a = _run(True, p, iters, memory, 2)
    from paper_2407_15049_b200 import alm
    alm.NATIVE_GENERIC = False
    try:
        b = _run(True, p, iters, memory, 2)
    finally:
        alm.NATIVE_GENERIC = True
    assert a[1] == b[1] and a[1] > 0
    assert a[0].tobytes() == b[0].tobytes()
    assert a[4].tobytes() == b[4].tobytes()
    assert a[2] == b[2] and a[3] == b[3]
    assert a[5] == b[5]

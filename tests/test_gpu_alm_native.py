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


def _run(native, p, iters, memory, seed, reduce_factor=None):
    import torch
    from paper_2407_15049_b200 import alm, linops
    from paper_2407_15049_b200.device import padded_ld
    alm.NATIVE = native
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
    admm.FUSED = False        # the one-launch step adds its sums in another order (test_gpu_admm_native.py)
    try:
        fast = driver.solve(p, cfg)
    finally:
        admm.FUSED = True
    tr = lambda rep: np.array([r[2:7] for r in rep.trace_rows], dtype=float)  # noqa: E731
    assert tr(fast).tobytes() == tr(slow).tobytes()
    assert fast.objective == slow.objective and fast.status == slow.status

"""Property tests of the device solve path, mirroring what the reference's own
unit tests establish (lrsdp tests/test_alm.py, test_admm.py, test_linops.py)
but re-derived against dense numpy linear algebra written here: operator
adjointness and positivity, the CG contract, half-step stationarity, fixed
points, gradients by finite differences, and the analytic optima of the
acceptance criteria (triangle 2.25, single edge 3, single observation 10).
Small and degenerate shapes on purpose: n = 1 (ld padding), m = 1, r = 1.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand_problem(rng, n, m, dens=0.3):
    from paper_2407_15049_b200.problem import SdpProblem, SymmetricSparse
    con, row, col, val = [], [], [], []
    for k in range(m):
        for i in range(n):
            for j in range(i, n):
                if rng.random() < dens:
                    con.append(k); row.append(i); col.append(j); val.append(float(rng.standard_normal()))
        if not con or con[-1] != k:
            con.append(k); row.append(k % n); col.append(k % n); val.append(1.0)
    ce = [(i, j, float(rng.standard_normal())) for i in range(n) for j in range(i, n) if rng.random() < dens]
    return SdpProblem(n=n, m=m, C=SymmetricSparse.from_entries(n, ce or [(0, 0, 1.0)]),
                      a_con=np.array(con), a_row=np.array(row), a_col=np.array(col), a_val=np.array(val),
                      b=rng.standard_normal(m))


def _dense(p):
    mats = []
    for k in range(p.m):
        A = np.zeros((p.n, p.n))
        sel = p.a_con == k
        A[p.a_row[sel], p.a_col[sel]] = p.a_val[sel]
        A[p.a_col[sel], p.a_row[sel]] = p.a_val[sel]
        mats.append(A)
    return mats, p.C.to_dense()


def _A(mats, X):
    return np.array([np.sum(M * X) for M in mats])


def _At(mats, y):
    return sum(yi * M for yi, M in zip(y, mats))


def _normal_matrix(mats, V, rho):
    """Dense matrix of W -> rho (A*(A(W V^T)) V + W) on vec(W) (column-major)."""
    n, r = V.shape
    M = np.zeros((n * r, n * r))
    for c in range(n * r):
        E = np.zeros(n * r)
        E[c] = 1.0
        W = E.reshape(n, r, order="F")
        M[:, c] = (rho * (_At(mats, _A(mats, W @ V.T)) @ V + W)).reshape(-1, order="F")
    return M


def test_subproblem_operator_self_adjoint_positive_and_dense():
    from paper_2407_15049_b200 import admm, linops
    rng = np.random.default_rng(21)
    for _ in range(12):
        n, m, r = int(rng.integers(1, 9)), int(rng.integers(1, 5)), int(rng.integers(1, 4))
        p = _rand_problem(rng, n, m)
        ops = linops.build_operators(p)
        mats, _ = _dense(p)
        rho = float(rng.uniform(0.2, 4.0))
        V, X, Y = (rng.standard_normal((n, r)) for _ in range(3))
        AX = admm.subproblem_apply(X, V, rho, ops)
        AY = admm.subproblem_apply(Y, V, rho, ops)
        assert abs(np.sum(AX * Y) - np.sum(AY * X)) <= 1e-11 * (1 + abs(np.sum(AX * Y)))
        assert np.sum(AX * X) >= rho * np.sum(X * X) - 1e-10
        want = (_normal_matrix(mats, V, rho) @ X.reshape(-1, order="F")).reshape(n, r, order="F")
        assert np.abs(AX - want).max() <= 1e-11 * (1 + np.abs(want).max())


def test_subproblem_rhs_matches_dense():
    from paper_2407_15049_b200 import admm, alm, linops
    rng = np.random.default_rng(22)
    for _ in range(10):
        n, m, r = int(rng.integers(1, 9)), int(rng.integers(1, 5)), int(rng.integers(1, 4))
        p = _rand_problem(rng, n, m)
        ops = linops.build_operators(p)
        mats, C = _dense(p)
        lam, rho, V = rng.standard_normal(m), float(rng.uniform(0.5, 3.0)), rng.standard_normal((n, r))
        want = (-C - _At(mats, lam) + rho * _At(mats, p.b)) @ V + rho * V
        got = admm.subproblem_rhs(V, alm.DualVector(lam, rho), ops)
        assert np.abs(got - want).max() <= 1e-11 * (1 + np.abs(want).max())


def test_cg_solves_the_half_step_system_and_is_stationary():
    from paper_2407_15049_b200 import admm, alm, linops
    rng = np.random.default_rng(23)
    for _ in range(6):
        n, m, r = int(rng.integers(2, 9)), int(rng.integers(1, 5)), 2
        p = _rand_problem(rng, n, m)
        ops = linops.build_operators(p)
        mats, C = _dense(p)
        rho, V, lam = float(rng.uniform(0.5, 3.0)), rng.standard_normal((n, r)), rng.standard_normal(m)
        rhs = admm.subproblem_rhs(V, alm.DualVector(lam, rho), ops)
        eps = 1e-12 * (1 + np.linalg.norm(rhs))
        x, its, res = admm.cg_solve(np.zeros((n, r)), lambda W: admm.subproblem_apply(W, V, rho, ops), rhs,
                                    admm.CgWorkspace(eps=eps, max_iter=n * r + 20))
        want = np.linalg.solve(_normal_matrix(mats, V, rho), rhs.reshape(-1, order="F")).reshape(n, r, order="F")
        assert np.abs(x - want).max() <= 1e-8 * (1 + np.abs(want).max())
        # stationarity of the coupled Lagrangian in U (admm.py docstring)
        g = C @ V + _At(mats, lam) @ V + rho * _At(mats, _A(mats, x @ V.T) - p.b) @ V + rho * (x - V)
        assert np.linalg.norm(g) <= 1e3 * eps


def test_cg_zero_iterations_at_solution_and_spd_violation():
    from paper_2407_15049_b200 import admm
    from paper_2407_15049_b200.exceptions import SpdViolationError
    rhs = np.ones((3, 1))
    x, its, res = admm.cg_solve(rhs / 3.0, lambda W: 3.0 * W, rhs, admm.CgWorkspace(eps=1e-10, max_iter=10))
    assert its == 0 and res <= 1e-10
    with pytest.raises(SpdViolationError):
        admm.cg_solve(np.zeros((2, 1)), lambda W: -W, np.ones((2, 1)), admm.CgWorkspace(eps=1e-12, max_iter=5))


def _scalar_problem(a=1.0, b=1.0):
    from paper_2407_15049_b200.problem import SdpProblem, SymmetricSparse
    return SdpProblem(n=1, m=1, C=SymmetricSparse.from_entries(1, []), a_con=np.array([0]),
                      a_row=np.array([0]), a_col=np.array([0]), a_val=np.array([a]), b=np.array([b]))


@pytest.mark.parametrize("native,fused", [(True, True), (True, False), (False, False)])
def test_admm_fixed_point_and_converged_start(native, fused):
    """n = m = 1 (a padded single column): a feasible complementary point stays put."""
    import torch
    from paper_2407_15049_b200 import admm, alm, linops
    p = _scalar_problem()
    ops = linops.build_operators(p)
    admm.NATIVE = native
    admm.FUSED = fused
    try:
        U = linops.to_factor(np.array([[1.0]]), ops.dev)
        st = admm.AdmmState(U=U.clone(), V=U.clone(), dual=alm.DualVector(lam=ops.dev.zeros(1), rho=2.0), r=1)
        admm.admm_step(st, ops)
        assert abs(float(st.U[0, 0]) - 1.0) <= 1e-10 and abs(float(st.V[0, 0]) - 1.0) <= 1e-10
        assert abs(float(st.dual.lam[0])) <= 1e-10
        assert float(torch.abs(st.U[:, 1:]).max()) == 0.0          # padding column stays zero
        res = admm.admm_run(st, ops, eps=1e-5, gap_eps=None)
        assert res.steps == 0
    finally:
        admm.NATIVE = True
        admm.FUSED = True


def test_alm_gradient_matches_finite_differences_and_value_matches_dense():
    from paper_2407_15049_b200 import alm, linops
    rng = np.random.default_rng(24)
    for _ in range(5):
        n, m, r = int(rng.integers(2, 7)), int(rng.integers(1, 4)), int(rng.integers(1, 3))
        p = _rand_problem(rng, n, m)
        ops = linops.build_operators(p)
        mats, C = _dense(p)
        lam, rho, scale = rng.standard_normal(m), float(rng.uniform(0.5, 2.0)), 0.6
        dual = alm.DualVector(lam, rho)

        def L(R):
            res = _A(mats, R @ R.T) - p.b
            return scale * np.sum(C * (R @ R.T)) + lam @ res + 0.5 * rho * res @ res
        R = rng.standard_normal((n, r))
        G = alm.alm_gradient(R, dual, ops, scale=scale)
        fd = np.zeros_like(R)
        h = 1e-6
        for i in range(n):
            for j in range(r):
                Rp, Rm = R.copy(), R.copy()
                Rp[i, j] += h
                Rm[i, j] -= h
                fd[i, j] = (L(Rp) - L(Rm)) / (2 * h)
        assert np.abs(G - fd).max() <= 1e-5 * (1 + np.abs(fd).max())
        assert abs(alm.alm_value(R, dual, ops, scale=scale) - L(R)) <= 1e-11 * (1 + abs(L(R)))


def test_line_search_quartic_reconstructs_the_lagrangian():
    from paper_2407_15049_b200 import alm, linops
    rng = np.random.default_rng(25)
    for _ in range(20):
        n, m, r = int(rng.integers(2, 7)), int(rng.integers(1, 4)), int(rng.integers(1, 3))
        p = _rand_problem(rng, n, m)
        ops = linops.build_operators(p)
        dual = alm.DualVector(rng.standard_normal(m), float(rng.uniform(0.5, 3.0)))
        R, D = rng.standard_normal((n, r)), rng.standard_normal((n, r))
        poly = alm.line_search_poly(R, D, dual, ops, scale=0.8)
        L0 = alm.alm_value(R, dual, ops, scale=0.8)
        for t in (-0.7, 0.3, 1.1):
            Lt = alm.alm_value(R + t * D, dual, ops, scale=0.8)
            assert abs((Lt - L0) - poly.value(t)) <= 1e-9 * (1 + abs(Lt))


def test_adjointness_and_maxcut_adjoint_of_ones():
    from paper_2407_15049_b200 import graphs, linops, problem
    rng = np.random.default_rng(26)
    for _ in range(10):
        n, m, r = int(rng.integers(1, 10)), int(rng.integers(1, 6)), int(rng.integers(1, 4))
        p = _rand_problem(rng, n, m)
        ops = linops.build_operators(p)
        U, V, y = rng.standard_normal((n, r)), rng.standard_normal((n, r)), rng.standard_normal(m)
        lhs = ops.cop.apply_pair(U, V) @ y
        S = ops.adj.assemble(lam=y, c_coeff=0.0)
        rhs = np.sum(linops.spmm(S, V) * U)
        assert abs(lhs - rhs) <= 1e-11 * (1 + abs(lhs))
    p = problem.build_maxcut(graphs.random_sparse(50, deg=4.0, seed=2))
    ops = linops.build_operators(p)
    X = rng.standard_normal((50, 3))
    assert np.abs(linops.spmm(ops.adj.assemble(lam=np.ones(50), c_coeff=0.0), X) - X).max() <= 1e-15


def test_dimension_mismatch_raises():
    from paper_2407_15049_b200 import linops
    from paper_2407_15049_b200.exceptions import DimensionMismatchError
    p = _rand_problem(np.random.default_rng(27), 5, 2)
    ops = linops.build_operators(p)
    with pytest.raises(DimensionMismatchError):
        ops.cop.apply_pair(np.zeros((5, 2)), np.zeros((4, 2)))
    with pytest.raises(DimensionMismatchError):
        ops.adj.apply(np.zeros(3))
    with pytest.raises(DimensionMismatchError):
        ops.cop.apply(np.zeros(ops.cop.ncols + 1))


@pytest.mark.parametrize("case,want,tol", [("triangle", 2.25, 1e-4), ("edge", 3.0, 1e-6),
                                           ("observation", 10.0, 1e-4)])
def test_analytic_optima(case, want, tol):
    """Acceptance criterion 2: triangle MaxCut 2.25, single edge 3, single observation 10."""
    from paper_2407_15049_b200 import driver, problem
    if case == "triangle":
        p = problem.build_maxcut(problem.GraphEdgeList.from_edges(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)]))
    elif case == "edge":
        p = problem.build_maxcut(problem.GraphEdgeList.from_edges(2, [(0, 1, 3.0)]))
    else:
        p = problem.build_matrix_completion(problem.ObservationSet.from_triples(1, 1, [(0, 0, 5.0)]))
    rep = driver.solve(p, driver.SolverConfig(reopt_level=2))
    assert rep.status == "optimal"
    assert abs(rep.objective - want) <= tol
    assert max(rep.err1, rep.err3, rep.err2) < 1e-5

"""Device operator layer vs the reference's golden outputs and the CPU oracle."""

import numpy as np
import pytest

from oracle import lrsdp_oracle as O
from tests._golden import load, ops_cases, problem_from

pytestmark = pytest.mark.gpu

TOL = 1e-12     # fp64, different summation order only


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / (1.0 + np.linalg.norm(b)))


@pytest.fixture(scope="module")
def P():
    import paper_2407_15049_b200 as P
    from paper_2407_15049_b200 import _lib
    _lib.load(require_device=True)
    return P


@pytest.mark.parametrize("case", ops_cases())
def test_operator_layer_matches_reference(P, case):
    from paper_2407_15049_b200 import admm, alm, linops
    z = load(f"ops_{case}.npz")
    p = problem_from(z)
    ops = linops.build_operators(p)
    U, V, D = z["U"], z["V"], z["D"]
    lam, extra, rho = z["lam"], z["extra"], float(z["rho"])
    assert ops.cop.ncols == int(z["K"])
    np.testing.assert_array_equal(ops.cop.imap.cpu().numpy(), z["imap"])
    np.testing.assert_array_equal(ops.cop.jmap.cpu().numpy(), z["jmap"])
    assert rel(ops.cop.outer_product(U, V), z["sddmm"]) <= TOL
    assert rel(ops.cop.apply_pair(U, V), z["AUV"]) <= TOL
    assert rel(ops.cop.apply(ops.cop.outer_product(U, V)), z["AUV"]) <= TOL
    S = ops.adj.assemble(lam=lam, extra=extra, c_coeff=-0.3)
    assert rel(S.toarray(), z["S_dense"]) <= TOL
    assert rel(linops.spmm(S, V), z["S_dense"] @ V) <= TOL
    dual = alm.DualVector(lam.copy(), rho)
    assert rel(alm.alm_gradient(U, dual, ops, scale=0.7), z["grad"]) <= TOL
    assert abs(alm.alm_value(U, dual, ops, scale=0.7) - float(z["value"])) <= TOL * (1 + abs(float(z["value"])))
    poly = alm.line_search_poly(U, D, dual, ops, scale=0.7)
    np.testing.assert_allclose(np.array(poly.coeffs()), z["poly"], rtol=1e-11, atol=1e-12)
    assert rel(poly.q1, z["q1"]) <= TOL and rel(poly.q2, z["q2"]) <= TOL
    assert rel(admm.subproblem_apply(U, V, rho, ops), z["half_apply"]) <= TOL
    rhs = admm.subproblem_rhs(V, dual, ops, scale=0.7)
    assert rel(rhs, z["half_rhs"]) <= TOL
    x, its, res = admm.cg_solve(np.zeros_like(U), lambda W: admm.subproblem_apply(W, V, rho, ops),
                                rhs, admm.CgWorkspace(eps=1e-9 * (1 + np.linalg.norm(rhs)), max_iter=50))
    assert abs(its - int(z["cg_its"])) <= 1
    assert rel(x, z["cg_x"]) <= 1e-9
    assert abs(ops.objective_value(U, V) - float(z["objective"])) <= TOL * (1 + abs(float(z["objective"])))


def test_lbfgs_direction_matches_two_loop(P):
    """Vector-free (Gram) L-BFGS direction == the reference's two-loop (alm.py:98)."""
    import torch
    from paper_2407_15049_b200 import alm
    from paper_2407_15049_b200.device import default_device
    z = load("lbfgs_linesearch.npz")
    dev = default_device()
    hist = alm.LbfgsHistory(8)
    bufs = []
    for s, y in zip(z["s"], z["y"]):
        sd = torch.as_tensor(s.reshape(-1)).cuda()
        yd = torch.as_tensor(y.reshape(-1)).cuda()
        bufs += [sd, yd]
        ys = float(np.sum(s * y))
        hist.push(sd, yd, 1.0, ys)
    g = torch.as_tensor(z["g"].reshape(-1)).cuda()
    allv = bufs + [g]
    for a in allv:
        for b in allv:
            hist.set_dot(a, b, float(torch.dot(a, b)))
    D = alm.lbfgs_direction(g, hist, dev)
    assert rel(D.cpu().numpy().reshape(z["D"].shape), z["D"]) <= 1e-12


def test_best_step_matches_reference_rule():
    from paper_2407_15049_b200 import alm
    z = load("lbfgs_linesearch.npz")
    for a, (t, zf) in zip(z["coeffs"], z["steps"]):
        tt, zz = alm.best_step(alm.LineSearchPoly(*[float(x) for x in a]))
        assert tt == t and float(zz) == zf


def test_lanczos_matches_reference(P):
    from paper_2407_15049_b200 import spectral
    z = load("spectral.npz")
    S = z["S"]
    est = spectral.smallest_eigenvalue(lambda v: S @ v, S.shape[0], seed=4)
    assert abs(est.value - float(z["value"])) <= 1e-10 * (1 + abs(float(z["value"])))
    assert est.basis_size == int(z["basis"])


@pytest.mark.parametrize("seed", range(20))
def test_random_fusion_equivalence_vs_oracle(P, seed):
    """A(U V^T), A*(y), assemble+SpMM, CG operator on random instances vs the oracle."""
    from paper_2407_15049_b200 import admm, linops
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 40))
    m = int(rng.integers(1, 10))
    r = int(rng.integers(1, 7))
    p = _random_problem(rng, n, m, r)
    ops = linops.build_operators(p)
    oo = O.OracleOps(p, dense_c=False)
    U = rng.standard_normal((n, r))
    V = rng.standard_normal((n, r))
    y = rng.standard_normal(m)
    assert rel(ops.cop.apply_pair(U, V), oo.A(U, V)) <= 1e-12
    assert rel(ops.adj.apply(y), oo.At_apply(y)) <= 1e-12
    S = ops.adj.assemble(lam=y, extra=2.0 * y, c_coeff=0.4)
    assert rel(linops.spmm(S, V), oo.assemble(lam=y, extra=2.0 * y, c_coeff=0.4) @ V) <= 1e-12
    assert rel(admm.subproblem_apply(U, V, 1.7, ops), O.half_apply(oo, U, V, 1.7)) <= 1e-12


def _random_problem(rng, n, m, r):
    from paper_2407_15049_b200.problem import SdpProblem, SymmetricSparse
    def sym(d):
        e = [(i, j, float(rng.standard_normal())) for i in range(n) for j in range(i, n)
             if rng.random() < d]
        return e or [(0, 0, 1.0)]
    con, row, col, val = [], [], [], []
    for k in range(m):
        for (i, j, v) in sym(min(0.3, 6.0 / n)):
            con.append(k); row.append(i); col.append(j); val.append(v)
    return SdpProblem(n=n, m=m, C=SymmetricSparse.from_entries(n, sym(0.2)),
                      a_con=np.array(con, dtype=np.int64), a_row=np.array(row, dtype=np.int64),
                      a_col=np.array(col, dtype=np.int64), a_val=np.array(val), b=rng.standard_normal(m))

"""Pin the CPU oracle (oracle/lrsdp_oracle.py) against the reference's own outputs.

The fixtures under tests/golden/ were produced by running the reference
package (tests/golden/make_golden.py). CPU only.
"""

import numpy as np
import pytest

from oracle import lrsdp_oracle as O
from tests._golden import cfg_of, load, ops_cases, problem_from, solve_cases


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / (1.0 + np.linalg.norm(b)))


@pytest.mark.parametrize("case", ops_cases())
def test_oracle_operator_layer_matches_reference(case):
    z = load(f"ops_{case}.npz")
    p = problem_from(z)
    dense = None if case == "random_densec" else False
    ops = O.OracleOps(p, dense_c=dense)
    U, V, D = z["U"], z["V"], z["D"]
    lam, extra, rho = z["lam"], z["extra"], float(z["rho"])
    assert ops.K == int(z["K"])
    assert len(ops.sup_i) == int(z["omega"])
    np.testing.assert_array_equal(ops.imap, z["imap"])
    np.testing.assert_array_equal(ops.jmap, z["jmap"])
    np.testing.assert_array_equal(ops.sddmm(U, V), z["sddmm"])
    np.testing.assert_array_equal(ops.A(U, V), z["AUV"])
    np.testing.assert_array_equal(ops.At_apply(lam), z["Aty"])
    S = ops.assemble(lam=lam, extra=extra, c_coeff=-0.3)
    S = S.toarray() if hasattr(S, "toarray") else S
    np.testing.assert_array_equal(S, z["S_dense"])
    ax = ops.A(U, U)
    np.testing.assert_array_equal(O.alm_grad(ops, U, lam, rho, 0.7, ax), z["grad"])
    CU = ops.c_mat @ U
    assert O.alm_val(ops, U, lam, rho, 0.7, ax, CU) == float(z["value"])
    a, q1, q2 = O.quartic(ops, U, D, lam, rho, 0.7, ax, CU, ops.c_mat @ D)
    np.testing.assert_array_equal(np.array(a), z["poly"])
    np.testing.assert_array_equal(O.half_apply(ops, U, V, rho), z["half_apply"])
    rhs = O.half_rhs(ops, V, lam, rho, 0.7)
    np.testing.assert_array_equal(rhs, z["half_rhs"])
    x, its, res = O.cg(np.zeros_like(U), lambda W: O.half_apply(ops, W, V, rho), rhs,
                       1e-9 * (1 + np.linalg.norm(rhs)), 50)
    assert its == int(z["cg_its"])
    np.testing.assert_array_equal(x, z["cg_x"])
    assert ops.objective(U, V) == float(z["objective"])


def test_oracle_lbfgs_and_step_rule_match_reference():
    z = load("lbfgs_linesearch.npz")
    pairs = []
    for s, y in zip(z["s"], z["y"]):
        O.push_pair(pairs, 8, s, y)
    np.testing.assert_array_equal(O.lbfgs_two_loop(z["g"], pairs), z["D"])
    for a, (t, zf) in zip(z["coeffs"], z["steps"]):
        tt, zz = O.step_length(tuple(float(x) for x in a))
        assert tt == t and float(zz) == zf


def test_oracle_lanczos_matches_reference():
    z = load("spectral.npz")
    S = z["S"]
    th, res, ok, k = O.min_eig(lambda v: S @ v, S.shape[0], seed=4)
    assert th == float(z["value"]) and k == int(z["basis"])
    assert abs(res - float(z["residual"])) <= 1e-12


@pytest.mark.parametrize("case", solve_cases())
def test_oracle_solve_trace_matches_reference(case):
    z = load(f"solve_{case}.npz")
    p = problem_from(z)
    out = O.solve(p, **cfg_of(z))
    tr = np.array([r[2:7] for r in out["trace"]], dtype=float).reshape(-1, 5)
    ref = z["trace"]
    assert out["status"] == str(z["status"])
    assert tr.shape == ref.shape
    # trace columns: objective, err1, metric, rho, rank
    np.testing.assert_allclose(tr, ref, rtol=1e-9, atol=1e-12)
    assert abs(out["objective"] - float(z["objective"])) <= 1e-9 * (1 + abs(float(z["objective"])))
    assert out["alm_inner"] == int(z["alm_inner"]) and out["admm_steps"] == int(z["admm_steps"])
    assert out["rank_history"] == list(z["rank_history"])

"""Parity at the bench's full size: BASELINE configs[2] (MaxCut, random sparse graph,
n = 10^7, average degree ~6, the solver's starting rank 25), the instance `bench.py` times.

The oracle cannot run whole operators at this size in test time, so parity is checked two
ways:

* sampled rows against the oracle: 4096 random rows of C X (linops.py:122 spmm with the
  objective), the ALM gradient (alm.py:239), the ADMM half-step operator and rhs
  (admm.py:45 / :52) and A(RR^T) (linops.py:70), each restated on those rows only from the
  oracle's symmetric CSR (`O.c_csr`, linops.py:197) and the diagonal constraints, to 1e-12
  relative (fp64, summation order only);
* size-independent identities over the whole instance: C symmetric (<U, CV> = <CU, V>),
  C linear, the ALM value equal to its definition from the device's own C R and A(RR^T)
  (alm.py:248), and the line-search quartic reproducing L(R + tD) - L(R) (alm.py:135).
"""

import math

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import lrsdp_oracle as O  # noqa: F401  (the restatement cited above)

pytestmark = pytest.mark.gpu

N, DEG, SEED, SAMPLE = 10_000_000, 6.0, 0, 4096


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / (1.0 + np.linalg.norm(b)))


@pytest.fixture(scope="module")
def full():
    from paper_2407_15049_b200 import _lib, driver, graphs, linops, problem
    _lib.load(require_device=True)
    p = problem.build_maxcut(graphs.random_sparse(N, deg=DEG, seed=SEED))
    assert np.array_equal(p.a_con, np.arange(p.m)) and np.array_equal(p.a_row, p.a_con)
    ops = linops.build_operators(p)
    r = driver.initial_rank(p.m, p.n)
    g = torch.Generator(device="cuda").manual_seed(1)
    X = [torch.randn(p.n, r, dtype=torch.float64, device="cuda", generator=g) / math.sqrt(p.n * r)
         for _ in range(3)]
    rows = np.sort(np.random.default_rng(2).choice(p.n, SAMPLE, replace=False))
    # the oracle's symmetric CSR of C (O.c_csr, linops.py:197), restricted to the sampled rows
    o = p.C.rows != p.C.cols
    rr = np.concatenate([p.C.rows, p.C.cols[o]])
    cc = np.concatenate([p.C.cols, p.C.rows[o]])
    vv = np.concatenate([p.C.vals, p.C.vals[o]])
    keep = np.isin(rr, rows)
    ucols, ci = np.unique(cc[keep], return_inverse=True)
    Cs = sp.csr_matrix((vv[keep], (np.searchsorted(rows, rr[keep]), ci)), shape=(SAMPLE, len(ucols)))
    return dict(p=p, ops=ops, r=r, X=X, rows=rows, ucols=ucols, Cs=Cs)


def _host_rows(T, idx):
    return T[torch.as_tensor(idx, device=T.device)].cpu().numpy()


def _c_rows(f, X):
    """Rows `f["rows"]` of C X, from the oracle CSR and X's referenced rows only."""
    return f["Cs"] @ _host_rows(X, f["ucols"])


def test_spmm_and_gradient_sampled_rows(full):
    from paper_2407_15049_b200 import alm, linops
    f = full
    p, ops, rows = f["p"], f["ops"], f["rows"]
    R = f["X"][0]
    CR = linops.spmm(ops.c_mat, R)
    assert rel(_host_rows(CR, rows), _c_rows(f, R)) <= 1e-12
    rng = np.random.default_rng(3)
    lam = 0.3 * rng.standard_normal(p.m)
    rho, scale = 7.5, 0.9
    ax = ops.cop.apply_pair(R, R)
    Rs = _host_rows(R, rows)
    a = p.a_val[rows]
    ax_s = a * np.einsum("ij,ij->i", Rs, Rs)                         # A(RR^T) on the sampled rows
    assert rel(_host_rows(ax.reshape(-1, 1), rows).ravel(), ax_s) <= 1e-13
    G = alm.alm_gradient(R, alm.DualVector(lam.copy(), rho), ops, scale=scale)
    w = lam[rows] + rho * (ax_s - p.b[rows])                       # alm.py:239: S = scale C + A*(w)
    want = 2.0 * (scale * _c_rows(f, R) + (a * w)[:, None] * Rs)
    assert rel(_host_rows(G, rows), want) <= 1e-12


def test_admm_operators_sampled_rows(full):
    from paper_2407_15049_b200 import admm, alm
    f = full
    p, ops, rows = f["p"], f["ops"], f["rows"]
    U, V = f["X"][0], f["X"][1]
    rho = 3.25
    out = admm.subproblem_apply(U, V, rho, ops)
    Us, Vs = _host_rows(U, rows), _host_rows(V, rows)
    a = p.a_val[rows]
    y = a * np.einsum("ij,ij->i", Us, Vs)                           # A(U V^T) on the sampled rows
    assert rel(_host_rows(out, rows), rho * ((a * y)[:, None] * Vs + Us)) <= 1e-12
    lam = np.random.default_rng(4).standard_normal(p.m)
    rhs = admm.subproblem_rhs(V, alm.DualVector(lam.copy(), rho), ops, scale=0.5)
    want = -0.5 * _c_rows(f, V) + (a * (rho * p.b[rows] - lam[rows]))[:, None] * Vs + rho * Vs
    assert rel(_host_rows(rhs, rows), want) <= 1e-12


def test_whole_instance_identities(full):
    from paper_2407_15049_b200 import alm, linops
    f = full
    p, ops = f["p"], f["ops"]
    U, V, D = f["X"]
    CU, CV = linops.spmm(ops.c_mat, U), linops.spmm(ops.c_mat, V)
    s1, s2 = float(torch.sum(U * CV)), float(torch.sum(CU * V))
    assert abs(s1 - s2) <= 1e-11 * (abs(s1) + float(torch.linalg.norm(CU) * torch.linalg.norm(V)))
    W = U + 2.0 * V
    CW = linops.spmm(ops.c_mat, W)
    assert float(torch.linalg.norm(CW - (CU + 2.0 * CV))) <= 1e-13 * float(torch.linalg.norm(CW)) * 4
    del CV, CW, W
    # alm.py:248 value from the device's own pieces, and the quartic (alm.py:135)
    R = U
    lam = torch.randn(p.m, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
    rho, scale = 5.0, 0.75
    dual = alm.DualVector(lam.cpu().numpy(), rho)
    res = ops.cop.apply_pair(R, R) - ops.b
    want = scale * float(torch.sum(CU * R)) + float(lam @ res) + 0.5 * rho * float(res @ res)
    L0 = alm.alm_value(R, dual, ops, scale=scale)
    assert abs(L0 - want) <= 1e-12 * (1.0 + abs(want))
    poly = alm.line_search_poly(R, D, dual, ops, scale=scale)
    for t in (-0.7, 0.3, 1.1):
        Lt = alm.alm_value(R + t * D, dual, ops, scale=scale)
        assert abs((Lt - L0) - poly.value(t)) <= 1e-9 * (1.0 + abs(Lt))

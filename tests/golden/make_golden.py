"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports lrsdp from /root/reference/pkg/src, draws seeded instances, runs
the reference's own operator-layer functions and full solves, and stores
inputs + outputs as small .npz files next to this script. The GPU box never
runs this script (it has no /root/reference); tests only read the .npz files.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from lrsdp import alm as ralm            # noqa: E402
from lrsdp import admm as radmm          # noqa: E402
from lrsdp import driver as rdrv         # noqa: E402
from lrsdp import linops as rlin         # noqa: E402
from lrsdp import problem as rprob       # noqa: E402
from lrsdp import spectral as rspec      # noqa: E402


def prob_arrays(p):
    return dict(n=p.n, m=p.m, c_rows=p.C.rows, c_cols=p.C.cols, c_vals=p.C.vals,
                a_con=p.a_con, a_row=p.a_row, a_col=p.a_col, a_val=p.a_val, b=p.b,
                maximize=p.maximize)


def random_problem(rng, n, m, density=0.3, c_density=0.3):
    """Seeded random symmetric-sparse SDP (same recipe as the reference's test oracle)."""
    def sym(d):
        e = [(i, j, float(rng.standard_normal())) for i in range(n) for j in range(i, n)
             if rng.random() < d]
        return e or [(0, 0, float(rng.standard_normal()))]
    con, row, col, val = [], [], [], []
    for k in range(m):
        for (i, j, v) in sym(density):
            con.append(k); row.append(i); col.append(j); val.append(v)
    C = rprob.SymmetricSparse.from_entries(n, sym(c_density))
    return rprob.SdpProblem(n=n, m=m, C=C, a_con=np.array(con, dtype=np.int64),
                            a_row=np.array(row, dtype=np.int64), a_col=np.array(col, dtype=np.int64),
                            a_val=np.array(val), b=rng.standard_normal(m))


def random_graph(rng, n, deg):
    """Uniform random simple graph with about n*deg/2 unit-weight edges."""
    me = int(n * deg / 2)
    u = rng.integers(0, n, size=int(me * 1.2) + 8)
    v = rng.integers(0, n, size=int(me * 1.2) + 8)
    a, b = np.minimum(u, v), np.maximum(u, v)
    keep = a != b
    code = np.unique(a[keep] * n + b[keep])
    code = np.sort(rng.permutation(code)[:me])
    return rprob.GraphEdgeList(n, code // n, code % n, np.ones(len(code)))


def lattice(side, rng):
    """Triangulated periodic lattice, random labels (Delaunay-like, degree 6)."""
    n = side * side
    i, j = np.divmod(np.arange(n), side)
    vid = lambda a, b: (a % side) * side + (b % side)  # noqa: E731
    u = np.concatenate([np.arange(n)] * 3)
    v = np.concatenate([vid(i, j + 1), vid(i + 1, j), vid(i + 1, j + 1)])
    perm = rng.permutation(n)
    u, v = perm[u], perm[v]
    a, b = np.minimum(u, v), np.maximum(u, v)
    code = np.unique(a * n + b)
    return rprob.GraphEdgeList(n, code // n, code % n, np.ones(len(code)))


def completion(rng, n2, n1, rank, frac):
    A = rng.standard_normal((n2, rank))
    B = rng.standard_normal((n1, rank))
    M = A @ B.T
    ii, jj = np.nonzero(rng.random((n2, n1)) < frac)
    return rprob.ObservationSet(n2, n1, ii.astype(np.int64), jj.astype(np.int64), M[ii, jj])


def operator_case(name, p, seed, r=3, dense_c=False):
    rng = np.random.default_rng(seed)
    ops = rlin.build_operators(p, dense_c=dense_c)
    n, m = p.n, p.m
    U = rng.standard_normal((n, r))
    V = rng.standard_normal((n, r))
    D = rng.standard_normal((n, r))
    lam = rng.standard_normal(m)
    extra = rng.standard_normal(m)
    rho = float(rng.uniform(0.5, 4.0))
    out = prob_arrays(p)
    dual = ralm.DualVector(lam.copy(), rho)
    ax = ops.cop.apply_pair(U, U)
    CU = rlin.spmm(ops.c_mat, U)
    CD = rlin.spmm(ops.c_mat, D)
    poly = ralm.line_search_poly(U, D, dual, ops, scale=0.7, ax=ax, CR=CU, CD=CD)
    S = ops.adj.assemble(lam=lam, extra=extra, c_coeff=-0.3)
    S = S.toarray() if hasattr(S, "toarray") else S
    rhs = radmm.subproblem_rhs(V, dual, ops, scale=0.7)
    ws = radmm.CgWorkspace(eps=1e-9 * (1 + np.linalg.norm(rhs)), max_iter=50)
    x, its, res = radmm.cg_solve(np.zeros((n, r)), lambda W: radmm.subproblem_apply(W, V, rho, ops),
                                 rhs, ws)
    out.update(
        U=U, V=V, D=D, lam=lam, extra=extra, rho=rho,
        K=ops.cop.ncols, omega=ops.adj.size, imap=ops.cop.imap, jmap=ops.cop.jmap,
        sddmm=ops.cop.outer_product(U, V), AUV=ops.cop.apply_pair(U, V),
        Aty=ops.adj.apply(lam), S_dense=S,
        grad=ralm.alm_gradient(U, dual, ops, scale=0.7),
        value=ralm.alm_value(U, dual, ops, scale=0.7),
        poly=np.array(poly.coeffs()), q1=poly.q1, q2=poly.q2,
        half_apply=radmm.subproblem_apply(U, V, rho, ops),
        half_rhs=rhs, cg_x=x, cg_its=its, cg_res=res,
        objective=ops.objective_value(U, V))
    np.savez_compressed(os.path.join(HERE, f"ops_{name}.npz"), **out)


def lbfgs_case():
    rng = np.random.default_rng(11)
    hist = ralm.LbfgsHistory(8)
    ss, ys = [], []
    while len(hist) < 6:
        s = rng.standard_normal((5, 3))
        y = s + 0.3 * rng.standard_normal((5, 3))
        if hist.push(s, y):
            ss.append(s); ys.append(y)
    g = rng.standard_normal((5, 3))
    D = ralm.lbfgs_direction(g, hist)
    coeffs = rng.standard_normal((200, 4)) * 3.0
    coeffs[:, 0] = np.abs(coeffs[:, 0])
    coeffs[50:60, 0] = 0.0
    coeffs[60:70, :2] = 0.0
    steps = []
    for a in coeffs:
        poly = ralm.LineSearchPoly(*a, p1=0, p2=0, q0=None, q1=None, q2=None)
        t, z = ralm.best_step(poly)
        steps.append((t, float(z)))
    np.savez_compressed(os.path.join(HERE, "lbfgs_linesearch.npz"), s=np.array(ss), y=np.array(ys),
                        g=g, D=D, coeffs=coeffs, steps=np.array(steps))


def spectral_case():
    rng = np.random.default_rng(12)
    n = 120
    A = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.05)
    S = A + A.T
    est = rspec.smallest_eigenvalue(lambda v: S @ v, n=n, seed=4)
    np.savez_compressed(os.path.join(HERE, "spectral.npz"), S=S, value=est.value,
                        residual=est.residual, basis=est.basis_size)


def _trace(rep):
    return np.array([r[2:7] for r in rep.trace_rows], dtype=np.float64).reshape(-1, 5)


def _first_dev(tr, ref, tol=1e-9):
    """First trace row where objective or err1 leaves the reference by > tol (relative)."""
    k = min(len(tr), len(ref))
    d = np.abs(tr[:k, 0] - ref[:k, 0]) / np.maximum(1.0, np.abs(ref[:k, 0]))
    e = np.abs(tr[:k, 1] - ref[:k, 1]) / (1e-4 + np.abs(ref[:k, 1]))
    bad = np.nonzero((d > tol) | (e > tol))[0]
    return int(bad[0]) if bad.size else k


def perturbed_runs(p, cfg, ref_trace, factors=(1.0, -1.0, 2.0, -2.0)):
    """Re-run the reference with its L-BFGS direction scaled by (1 + f*2^-52).

    The reference is chaotic: a one-ulp change of one vector moves later
    iterates. The spread of these runs is the reference's own reproducibility
    envelope, against which the device solver is judged.
    """
    orig = ralm.lbfgs_direction
    out = []
    try:
        for f in factors:
            scale = 1.0 + f * 2.0 ** -52
            ralm.lbfgs_direction = lambda g, h, _s=scale: orig(g, h) * _s
            rep = rdrv.solve(p, rdrv.SolverConfig(**cfg))
            out.append((_first_dev(_trace(rep), ref_trace), rep.objective, len(rep.trace_rows),
                        rep.status))
    finally:
        ralm.lbfgs_direction = orig
    return out


def solve_case(name, p, **cfg):
    rep = rdrv.solve(p, rdrv.SolverConfig(**cfg))
    out = prob_arrays(p)
    pert = perturbed_runs(p, cfg, _trace(rep))
    out.update(ulp_horizon=np.array([x[0] for x in pert]), ulp_objective=np.array([x[1] for x in pert]),
               ulp_rows=np.array([x[2] for x in pert]), ulp_status=np.array([x[3] for x in pert]))
    tr = np.array([r[2:7] for r in rep.trace_rows], dtype=np.float64).reshape(-1, 5)
    stage = np.array([0 if r[0] == "alm" else 1 for r in rep.trace_rows], dtype=np.int8)
    out.update(trace=tr, trace_stage=stage, objective=rep.objective, err1=rep.err1,
               err2=rep.err2 if rep.err2 is not None else np.nan, err3=rep.err3,
               rank_history=np.array(rep.rank_history), reopt_rounds=rep.reopt_rounds,
               alm_outer=rep.alm_outer_iterations, alm_inner=rep.alm_inner_iterations,
               admm_steps=rep.admm_steps, cg=rep.cg_iterations, K=rep.K, omega=rep.omega_size,
               status=rep.status, cfg=json.dumps(cfg))
    np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), **out)
    print(name, rep.status, rep.objective, rep.err1, rep.err2, rep.err3, rep.rank_history,
          rep.alm_inner_iterations, rep.admm_steps, rep.reopt_rounds, rep.time_total_s,
          "ulp:", pert, flush=True)


def main():
    rng = np.random.default_rng(2024)
    operator_case("random_sparse", random_problem(rng, 14, 6, density=0.2, c_density=0.2), 1)
    operator_case("random_densec", random_problem(rng, 9, 4, density=0.4, c_density=0.9), 2,
                  dense_c=None)
    operator_case("maxcut_g60", rprob.build_maxcut(random_graph(rng, 60, 5)), 3, r=4)
    operator_case("completion", rprob.build_matrix_completion(completion(rng, 7, 6, 2, 0.5)), 4)
    lbfgs_case()
    spectral_case()
    tri = rprob.build_maxcut(rprob.GraphEdgeList.from_edges(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)]))
    solve_case("triangle_l2", tri, reopt_level=2)
    solve_case("single_edge", rprob.build_maxcut(rprob.GraphEdgeList.from_edges(2, [(0, 1, 3.0)])))
    solve_case("g1_like", rprob.build_maxcut(random_graph(np.random.default_rng(1), 800, 48)))
    solve_case("maxcut_2k_deg6", rprob.build_maxcut(random_graph(np.random.default_rng(2), 2000, 6)),
               admm_step_cap=1500, max_reopts=0)
    solve_case("delaunay_45", rprob.build_maxcut(lattice(45, np.random.default_rng(5))),
               admm_step_cap=1500, max_reopts=1)
    solve_case("completion_30", rprob.build_matrix_completion(
        completion(np.random.default_rng(3), 30, 30, 2, 0.4)))
    solve_case("random_sdp", random_problem(np.random.default_rng(4), 10, 5, density=0.3,
                                            c_density=0.3), reopt_level=0)


if __name__ == "__main__":
    main()

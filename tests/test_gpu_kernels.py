"""Edge cases of the sm_100a kernels against plain numpy/scipy references.

Targets the paths the golden instances do not reach: tiles whose staged
segment overflows shared memory (dense rows), empty rows, row counts that are
not a multiple of the tile, every lane-group width (ld 1 .. 130, including
ranks above 64 where a row is processed in column chunks), the assembled-
coefficient SpMM, the diagonal-constraint fast path and every history-width
bucket of the fused ALM update.
"""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2407_15049_b200 import _lib
    from paper_2407_15049_b200.device import default_device
    _lib.load(require_device=True)
    return default_device()


def _pattern(M, at=None):
    """DevicePattern of a scipy CSR (values as cv); optional adjoint rows (at_ptr, at_con, at_val)."""
    import torch
    from paper_2407_15049_b200.linops import DevicePattern, padded
    M = sp.csr_matrix(M)
    M.sort_indices()
    c = lambda a, dt: padded(torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dt))  # noqa: E731
    ptr = c(M.indptr.astype(np.int64), torch.int64)
    idx = c(M.indices.astype(np.int32), torch.int32)
    cv = c(M.data.astype(np.float64), torch.float64)
    if at is None:
        return DevicePattern(M.shape[0], ptr, idx, cv, None, None, None)
    ap, ac, av = at
    return DevicePattern(M.shape[0], ptr, idx, cv, c(ap, torch.int64), c(ac, torch.int32),
                         c(av, torch.float64))


def _rand_csr(rng, n, ncols, deg_fn):
    rows, cols = [], []
    for i in range(n):
        d = deg_fn(i)
        cs = np.unique(rng.integers(0, ncols, size=d)) if d else np.zeros(0, dtype=np.int64)
        rows += [i] * len(cs)
        cols += list(cs)
    vals = rng.standard_normal(len(rows))
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, ncols))


def _factor(rng, n, ld):
    import torch
    X = rng.standard_normal((n, ld))
    return X, torch.as_tensor(X).cuda().contiguous()


@pytest.mark.parametrize("ld", [1, 2, 4, 6, 16, 26, 30, 66, 130])
@pytest.mark.parametrize("shape", ["sparse", "dense_rows", "empty_rows"])
def test_tiled_spmm_matches_scipy(dev, ld, shape):
    import torch
    rng = np.random.default_rng(ld * 7 + len(shape))
    n = 3001
    if shape == "sparse":
        M = _rand_csr(rng, n, n, lambda i: int(rng.integers(0, 12)))
    elif shape == "dense_rows":       # rows far longer than one staged tile (> 1024 slots)
        M = _rand_csr(rng, n, n, lambda i: 1500 if i % 97 == 0 else int(rng.integers(1, 8)))
    else:
        M = _rand_csr(rng, n, n, lambda i: 0 if i % 3 else int(rng.integers(1, 30)))
    P = _pattern(M)
    X, Xd = _factor(rng, n, ld)
    out = torch.empty_like(Xd)
    dev.spmm(P, Xd, ld, alpha=0.75, out=out, c_coeff=-1.5)
    ref = 0.75 * (-1.5) * (M @ X)
    err = np.abs(out.cpu().numpy() - ref).max() / (1 + np.abs(ref).max())
    assert err <= 1e-13, err


@pytest.mark.parametrize("ld", [1, 6, 26, 66])
def test_tiled_spmm_epilogue_and_dots(dev, ld):
    import torch
    rng = np.random.default_rng(5 + ld)
    n = 2000
    M = _rand_csr(rng, n, n, lambda i: int(rng.integers(1, 9)))
    P = _pattern(M)
    X, Xd = _factor(rng, n, ld)
    Y, Yd = _factor(rng, n, ld)
    Z, Zd = _factor(rng, n, ld)
    out = torch.empty_like(Xd)
    dev.spmm(P, Xd, ld, alpha=2.0, out=out, Y=[Yd], ycoef=[-0.5], Z=[Zd],
             dots=[("out", "out"), ("out", ("z", 0)), (("y", 0), ("z", 0))], at=10, c_coeff=1.0)
    s = dev.fetch(13)[10:13]
    o = 2.0 * (M @ X) - 0.5 * Y
    assert np.abs(out.cpu().numpy() - o).max() <= 1e-12 * (1 + np.abs(o).max())
    for got, want in zip(s, [np.sum(o * o), np.sum(o * Z), np.sum(Y * Z)]):
        assert abs(got - want) <= 1e-11 * (1 + abs(want))


def test_assembled_coefficient_spmm(dev):
    """S = c*C + A*(w1) + A*(w2) assembled into scratch, then the tiled product."""
    import torch
    rng = np.random.default_rng(9)
    n, m = 1500, 400
    M = _rand_csr(rng, n, n, lambda i: int(rng.integers(1, 10)))
    nnz = M.nnz
    # each slot gets 0..3 adjoint entries
    cnt = rng.integers(0, 4, size=nnz)
    at_ptr = np.zeros(nnz + 1, dtype=np.int64)
    at_ptr[1:] = np.cumsum(cnt)
    at_con = rng.integers(0, m, size=at_ptr[-1]).astype(np.int32)
    at_val = rng.standard_normal(at_ptr[-1])
    P = _pattern(M, (at_ptr, at_con, at_val))
    w1, w2 = rng.standard_normal(m), rng.standard_normal(m)
    coef = np.array([np.dot(at_val[at_ptr[s]:at_ptr[s + 1]], w1[at_con[at_ptr[s]:at_ptr[s + 1]]])
                     + np.dot(at_val[at_ptr[s]:at_ptr[s + 1]], w2[at_con[at_ptr[s]:at_ptr[s + 1]]])
                     for s in range(nnz)]) + 0.3 * sp.csr_matrix(M).data
    S = sp.csr_matrix((coef, M.indices, M.indptr), shape=M.shape)
    X, Xd = _factor(rng, n, 26)
    out = torch.empty_like(Xd)
    dev.spmm(P, Xd, 26, out=out, c_coeff=0.3, w1=torch.as_tensor(w1).cuda(), w2=torch.as_tensor(w2).cuda())
    ref = S @ X
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * (1 + np.abs(ref).max())


@pytest.mark.parametrize("ld", [2, 26, 66, 130, 4098])
def test_diag_constraint_fast_path_equals_generic(dev, ld):
    """cl_diag_constraint_eval and cl_constraint_eval agree on diagonal constraints (summation order differs)."""
    import torch
    from paper_2407_15049_b200 import graphs, linops, problem
    p = problem.build_maxcut(graphs.random_sparse(5000, deg=6.0, seed=ld))
    ops = linops.build_operators(p)
    con = ops.cop.con
    assert con.diag_aval is not None
    rng = np.random.default_rng(ld)
    X = [torch.as_tensor(rng.standard_normal((p.n, ld))).cuda() for _ in range(6)]
    o_fast = [torch.empty(p.m, dtype=torch.float64, device="cuda") for _ in range(2)]
    o_gen = [torch.empty(p.m, dtype=torch.float64, device="cuda") for _ in range(2)]
    dev.constraint_eval(con, ld, X[0], X[1], o_fast[0], X2=X[2], Y2=X[3], X3=X[4], Y3=X[5], out2=o_fast[1])
    saved, con.diag_aval = con.diag_aval, None
    try:
        dev.constraint_eval(con, ld, X[0], X[1], o_gen[0], X2=X[2], Y2=X[3], X3=X[4], Y3=X[5], out2=o_gen[1])
    finally:
        con.diag_aval = saved
    for a, b in zip(o_fast, o_gen):
        a, b = a.cpu().numpy(), b.cpu().numpy()
        assert np.abs(a - b).max() <= 1e-14 * (1 + np.abs(b).max())
    Xh = [x.cpu().numpy() for x in X]
    want = np.einsum("ij,ij->i", Xh[0], Xh[1]) + np.einsum("ij,ij->i", Xh[2], Xh[3])
    assert np.abs(o_fast[0].cpu().numpy() - want).max() <= 1e-12 * (1 + np.abs(want).max())


@pytest.mark.parametrize("nh", [0, 3, 9, 17])
@pytest.mark.parametrize("refresh", [True, False])
def test_diag_alm_update_buckets(dev, nh, refresh):
    import torch
    from paper_2407_15049_b200 import _lib
    rng = np.random.default_rng(nh + 100 * refresh)
    n, ld = 3000, 26
    T = lambda *s: torch.as_tensor(rng.standard_normal(s)).cuda().contiguous()  # noqa: E731
    R, D, CR, CD, gold = T(n, ld), T(n, ld), T(n, ld), T(n, ld), T(n, ld)
    ax, q1, q2, lam, b, aval = T(n), T(n), T(n), T(n), T(n), T(n)
    H = [T(n, ld) for _ in range(nh)]
    gnew, y = torch.empty_like(R), torch.empty_like(R)
    axo = torch.empty_like(ax)
    tau, rho, scale = 0.37, 2.5, 0.8
    Rh, Dh, CRh, CDh, goh = [t.cpu().numpy() for t in (R, D, CR, CD, gold)]
    axh, q1h, q2h, lamh, bh, ah = [t.cpu().numpy() for t in (ax, q1, q2, lam, b, aval)]
    Hh = [h.cpu().numpy() for h in H]
    a = _lib.DiagUpdateArgs()
    a.n, a.ld, a.aval = n, ld, aval.data_ptr()
    a.tau, a.rho, a.scale = tau, rho, scale
    a.R, a.D, a.CR, a.CD = R.data_ptr(), D.data_ptr(), CR.data_ptr(), CD.data_ptr()
    a.ax, a.ax_out, a.q1, a.q2 = ax.data_ptr(), axo.data_ptr(), q1.data_ptr(), q2.data_ptr()
    a.lam, a.b, a.g_old, a.g_new, a.y = lam.data_ptr(), b.data_ptr(), gold.data_ptr(), gnew.data_ptr(), y.data_ptr()
    a.nh = nh
    for j, h in enumerate(H):
        a.H[j] = h.data_ptr()
    a.refresh = 1 if refresh else 0
    dev.diag_update(a, at=0)
    s = dev.fetch(7 + 2 * _lib.CL_MAXIN)
    if not refresh:
        Rh = Rh + tau * Dh
        CRh = CRh + tau * CDh
        axh = axh + tau * q1h + tau * tau * q2h
    res = axh - bh
    w = lamh + rho * res
    g = 2.0 * ((w * ah)[:, None] * Rh + scale * CRh)
    yy = g - goh
    close = lambda u, v: abs(u - v) <= 1e-10 * (1 + abs(v))  # noqa: E731
    assert np.abs(gnew.cpu().numpy() - g).max() <= 1e-12 * (1 + np.abs(g).max())
    assert close(s[0], np.sum(CRh * Rh)) and close(s[1], np.sum(g * g)) and close(s[2], np.sum(yy * Dh))
    assert close(s[3], np.dot(lamh, res)) and close(s[4], np.dot(res, res))
    for h in range(nh):
        assert close(s[7 + h], np.sum(g * Hh[h]))
        assert close(s[7 + _lib.CL_MAXIN + h], np.sum(yy * Hh[h]))


class _FakeHalo:
    """Stands in for shard.HaloPlan: columns >= nown read a fixed ghost block."""

    def __init__(self, nown, ghost):
        self.nown, self.ghost, self.calls = nown, ghost, 0

    def exchange(self, X, ld, pack):
        self.calls += 1
        return self.ghost


@pytest.mark.parametrize("ld", [2, 26, 66])
def test_ghost_rows_in_tiled_spmm(dev, ld):
    """Row-sharded SpMM: column j < nown reads the local factor, j >= nown the halo block."""
    import torch
    rng = np.random.default_rng(40 + ld)
    nown, nghost = 2500, 1700
    M = _rand_csr(rng, nown, nown + nghost, lambda i: int(rng.integers(0, 14)))
    P = _pattern(M)
    Xo, Xod = _factor(rng, nown, ld)
    Xg, Xgd = _factor(rng, nghost, ld)
    P.halo = _FakeHalo(nown, Xgd)
    out = torch.empty_like(Xod)
    dev.spmm(P, Xod, ld, out=out, c_coeff=1.0, Z=[Xod], dots=[("out", ("z", 0))], at=20)
    ref = M @ np.vstack([Xo, Xg])
    assert P.halo.calls == 1
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * (1 + np.abs(ref).max())
    assert abs(dev.fetch(21)[20] - np.sum(ref * Xo)) <= 1e-10 * (1 + abs(np.sum(ref * Xo)))


def test_gather_rows_kernel(dev):
    import torch
    rng = np.random.default_rng(3)
    X, Xd = _factor(rng, 1000, 26)
    idx = rng.choice(1000, size=321, replace=False).astype(np.int32)
    out = torch.zeros((400, 26), dtype=torch.float64, device="cuda")
    dev.gather_rows(torch.as_tensor(idx).cuda(), Xd, out)
    got = out.cpu().numpy()
    assert np.array_equal(got[:321], X[idx]) and not got[321:].any()


@pytest.mark.parametrize("r", [1, 5, 13, 30])
def test_single_entry_apply_matches_generic_operator(dev, r):
    """Matrix completion's constraints are single-entry: the fused half-step operator
    (cl_single_entry_apply) equals constraint pass + assembled SpMM."""
    import torch
    from paper_2407_15049_b200 import admm, graphs, linops, problem
    from paper_2407_15049_b200.device import padded_ld
    p = problem.build_matrix_completion(graphs.random_completion(300, 250, 6000, seed=r))
    ops = linops.build_operators(p)
    assert ops.adj.apat.single_a is not None and not ops.is_diag
    ld = padded_ld(r)
    rng = np.random.default_rng(r)
    W = linops.to_factor(rng.standard_normal((p.n, r)), dev, ld)
    Wf = linops.to_factor(rng.standard_normal((p.n, r)), dev, ld)
    hs = admm.HalfStep(ops, p.n, ld)
    fused = torch.empty_like(W)
    hs.apply(W, Wf, 1.7, fused, dot_with=W, at=30)
    d_fused = dev.fetch(31)[30]
    saved, ops.adj.apat.single_a = ops.adj.apat.single_a, None
    try:
        gen = torch.empty_like(W)
        hs.apply(W, Wf, 1.7, gen, dot_with=W, at=30)
        d_gen = dev.fetch(31)[30]
    finally:
        ops.adj.apat.single_a = saved
    f, g = fused.cpu().numpy(), gen.cpu().numpy()
    # same row dots, same association, same slot order: bit-identical operators
    assert f.tobytes() == g.tobytes()
    assert abs(d_fused - d_gen) <= 1e-12 * (1 + abs(d_gen))


@pytest.mark.parametrize("r", [3, 8, 25, 50])
def test_single_entry_pair_buffer_bit_identical(dev, r):
    """cl_single_entry_apply_pair on the pair buffer [W | Wf] (cl_pair_pack) equals the
    two-operand kernel bit for bit, output and <W, out>; cl_cg_direction_pair equals the
    lincomb p = r + beta p and mirrors it into the pair buffer."""
    import torch
    from paper_2407_15049_b200 import admm, graphs, linops, problem
    from paper_2407_15049_b200.device import padded_ld
    p = problem.build_matrix_completion(graphs.random_completion(400, 350, 9000, seed=r))
    ops = linops.build_operators(p)
    apat = ops.adj.apat
    ld = padded_ld(r)
    rng = np.random.default_rng(r)
    W = linops.to_factor(rng.standard_normal((p.n, r)), dev, ld)
    Wf = linops.to_factor(rng.standard_normal((p.n, r)), dev, ld)
    a, b = torch.empty_like(W), torch.empty_like(W)
    dev.single_entry_apply(apat, ld, W, Wf, 1.3, a, at=30)
    da = float(dev.fetch(31)[30])
    P2 = dev.empty(p.n, 2 * ld)
    dev.pair_pack(W, ld, P2, 0)
    dev.pair_pack(Wf, ld, P2, 1)
    assert torch.equal(P2[:, :ld], W) and torch.equal(P2[:, ld:], Wf)
    dev.single_entry_apply_pair(apat, ld, P2, 1.3, b, at=30)
    db = float(dev.fetch(31)[30])
    assert a.cpu().numpy().tobytes() == b.cpu().numpy().tobytes() and da == db
    rr = linops.to_factor(rng.standard_normal((p.n, r)), dev, ld)
    p1, p2 = W.clone(), W.clone()
    dev.lincomb(p1, [rr, p1], [1.0, 0.37])
    dev.cg_direction_pair(ld, 0.37, rr, p2, P2)
    assert torch.equal(p1, p2) and torch.equal(P2[:, :ld], p2) and torch.equal(P2[:, ld:], Wf)


def test_pair_cg_matches_two_operand_cg(dev):
    """A whole completion half-step CG on the pair buffer: the same iterates, residuals and
    iteration count as the two-operand path (admm.PAIR off)."""
    from paper_2407_15049_b200 import admm, alm, graphs, linops, problem
    from paper_2407_15049_b200.device import padded_ld
    p = problem.build_matrix_completion(graphs.random_completion(500, 400, 12000, seed=9))
    ops = linops.build_operators(p)
    r = 12
    ld = padded_ld(r)
    rng = np.random.default_rng(3)
    U = linops.to_factor(rng.standard_normal((p.n, r)) / 20, dev, ld)
    V = linops.to_factor(rng.standard_normal((p.n, r)) / 20, dev, ld)
    out = []
    for pair in (True, False):
        admm.PAIR = pair
        try:
            st = admm.AdmmState(U=U.clone(), V=V.clone(), dual=alm.DualVector(lam=dev.zeros(p.m), rho=2.0), r=r)
            hs = admm.HalfStep(ops, p.n, ld)
            stats = [admm.admm_step(st, ops, hs=hs) for _ in range(3)]
        finally:
            admm.PAIR = True
        out.append((st.U.cpu().numpy(), st.V.cpu().numpy(), [(s.cg_iters_u, s.cg_iters_v, s.resid_u, s.resid_v)
                                                             for s in stats]))
    (u1, v1, s1), (u2, v2, s2) = out
    assert sum(a + b for a, b, _, _ in s1) > 0          # the CGs iterate
    assert s1 == s2 and u1.tobytes() == u2.tobytes() and v1.tobytes() == v2.tobytes()


@pytest.mark.parametrize("r", [3, 25, 50])
def test_constraint_eval_pair_bit_identical(dev, r):
    """cl_constraint_eval_pair on [R | D] equals the line search's three-product
    cl_constraint_eval (X1=R, Y1=D, X2=D, Y2=R, X3=Y3=D) bit for bit."""
    from paper_2407_15049_b200 import graphs, linops, problem
    from paper_2407_15049_b200.device import padded_ld
    p = problem.build_matrix_completion(graphs.random_completion(300, 260, 7000, seed=r))
    ops = linops.build_operators(p)
    con = ops.cop.con
    ld = padded_ld(r)
    rng = np.random.default_rng(r)
    R = linops.to_factor(rng.standard_normal((p.n, r)), dev, ld)
    D = linops.to_factor(rng.standard_normal((p.n, r)), dev, ld)
    q1, q2, s1, s2 = dev.empty(p.m), dev.empty(p.m), dev.empty(p.m), dev.empty(p.m)
    dev.constraint_eval(con, ld, R, D, q1, X2=D, Y2=R, X3=D, Y3=D, out2=q2)
    P2 = dev.empty(p.n, 2 * ld)
    dev.pair_pack(R, ld, P2, 0)
    dev.pair_pack(D, ld, P2, 1)
    dev.constraint_eval_pair(con, ld, P2, s1, s2)
    assert q1.cpu().numpy().tobytes() == s1.cpu().numpy().tobytes()
    assert q2.cpu().numpy().tobytes() == s2.cpu().numpy().tobytes()


def test_pair_line_search_alm_matches(dev):
    """A completion ALM inner solve with the pair-buffer line search (alm.PAIR) follows
    the two-operand line search bit for bit."""
    from paper_2407_15049_b200 import alm, graphs, linops, problem
    from paper_2407_15049_b200.device import padded_ld
    p = problem.build_matrix_completion(graphs.random_completion(400, 300, 9000, seed=4))
    ops = linops.build_operators(p)
    r = 10
    ld = padded_ld(r)
    R0 = linops.to_factor(np.random.default_rng(1).standard_normal((p.n, r)) / 10, dev, ld)
    out = []
    for pair in (True, False):
        alm.PAIR = pair
        try:
            core = alm.AlmCore(ops, p.n, ld)
            R = R0.clone()
            res = alm._inner(core, R, dev.zeros(p.m), 3.0, 1.0, 0.0, 25, None, 8, alm._RankRecorder(None, r))
        finally:
            alm.PAIR = True
        out.append((R.cpu().numpy(), res.iterations, res.grad_norms))
    assert out[0][1] == out[1][1] > 0 and out[0][2] == out[1][2]
    assert out[0][0].tobytes() == out[1][0].tobytes()


def test_single_entry_detection_rejects_general_constraints(dev):
    from paper_2407_15049_b200 import linops
    from tests._golden import load, problem_from
    ops = linops.build_operators(problem_from(load("solve_random_sdp.npz")))
    assert ops.adj.apat.single_a is None


@pytest.mark.parametrize("case", ["maxcut", "completion", "tiny", "breakdown"])
def test_native_lanczos_bit_identical(dev, case):
    """cl_lanczos_loop (operator assembled once, CL_LANCZOS_BATCH steps per round trip) vs
    the Python-driven loop: same eigenvalue estimate to the bit, and the same basis size;
    also for a basis smaller than one batch (tiny) and a Krylov breakdown inside a batch
    (complete graph, constant multiplier: C - A*(lam) has two distinct eigenvalues)."""
    from paper_2407_15049_b200 import graphs, linops, problem, spectral
    lam = None
    if case == "maxcut":
        p = problem.build_maxcut(graphs.random_sparse(700, deg=8.0, seed=5))
    elif case == "tiny":
        p = problem.build_maxcut(graphs.GraphEdgeList(3, np.array([0, 1]), np.array([1, 2]), np.ones(2)))
    elif case == "breakdown":
        n = 40
        iu, ju = np.triu_indices(n, 1)
        p = problem.build_maxcut(graphs.GraphEdgeList(n, iu, ju, np.ones(iu.size)))
        lam = np.full(p.m, 0.3)
    else:
        p = problem.build_matrix_completion(graphs.random_completion(60, 50, 900, seed=5))
    ops = linops.build_operators(p)
    if lam is None:
        lam = np.random.default_rng(7).standard_normal(p.m)
    res = {}
    for native in (True, False):
        spectral.NATIVE = native
        spectral.FUSED = False
        try:
            res[native] = spectral.dual_infeasibility(p, ops, lam, tol=1e-7, seed=3)
        finally:
            spectral.NATIVE = True
            spectral.FUSED = True
    assert res[True] == res[False]
    # the one-launch loop (cl_lanczos_loop_fused): the same estimate to rounding
    fused = spectral.dual_infeasibility(p, ops, lam, tol=1e-7, seed=3)
    assert fused[1] == res[True][1]
    for u, v in ((fused[0], res[True][0]), (fused[2], res[True][2])):
        assert abs(u - v) <= 1e-9 * (1.0 + abs(v))


@pytest.mark.parametrize("ld", [2, 26, 66, 130])
def test_fused_admm_passes_match_numpy(dev, ld):
    """cl_diag_admm_cg_init / cl_diag_admm_step_end against dense numpy, including ranks
    whose rows span several column chunks."""
    import torch
    from paper_2407_15049_b200 import graphs, linops, problem
    p = problem.build_maxcut(graphs.random_sparse(1500, deg=7.0, seed=ld))
    ops = linops.build_operators(p)
    rng = np.random.default_rng(ld)
    T = lambda *s: torch.as_tensor(rng.standard_normal(s)).cuda().contiguous()  # noqa: E731
    Wf, x0, U, V = T(p.n, ld), T(p.n, ld), T(p.n, ld), T(p.n, ld)
    nlam, lam = T(p.m), T(p.m)
    aval = ops.diag_aval
    r = torch.empty_like(Wf)
    scale, rho = 0.7, 1.9
    dev.diag_admm_cg_init(ops.c_mat.cpat, Wf, x0, ld, scale, rho, nlam, aval, r, at=60)
    ax = torch.empty(p.m, dtype=torch.float64, device="cuda")
    lam_new = torch.empty_like(ax)
    dev.diag_admm_step_end(ops.c_mat.cpat, U, V, ld, aval, ops.b, lam, rho, ax, lam_new, at=62)
    s = dev.fetch(65)
    C = sp.csr_matrix((ops.c_mat.cpat.cv.cpu().numpy(), ops.c_mat.cpat.indices.cpu().numpy(),
                       ops.c_mat.cpat.indptr.cpu().numpy()), shape=(p.n, p.n))
    a = aval.cpu().numpy()
    Wh, xh, Uh, Vh = [t.cpu().numpy() for t in (Wf, x0, U, V)]
    rhs = -scale * (C @ Wh) + rho * Wh + (a * nlam.cpu().numpy())[:, None] * Wh
    y = a * np.einsum("ij,ij->i", xh, Wh)
    Q = rho * ((a * y)[:, None] * Wh + xh)
    rr = rhs - Q
    close = lambda u, v, t=1e-11: abs(u - v) <= t * (1 + abs(v))  # noqa: E731
    assert np.abs(r.cpu().numpy() - rr).max() <= 1e-11 * (1 + np.abs(rr).max())
    assert close(s[60], np.sum(rhs * rhs)) and close(s[61], np.sum(rr * rr))
    axh = a * np.einsum("ij,ij->i", Uh, Vh)
    res = axh - ops.b.cpu().numpy()
    ln = lam.cpu().numpy() + rho * res
    assert np.abs(ax.cpu().numpy() - axh).max() <= 1e-11 * (1 + np.abs(axh).max())
    assert np.abs(lam_new.cpu().numpy() - ln).max() <= 1e-11 * (1 + np.abs(ln).max())
    assert close(s[62], np.sum((C @ Vh) * Uh)) and close(s[63], res @ res)
    assert close(s[64], ln @ ops.b.cpu().numpy())
    # the stored C Wf and the streaming step end built on it (cl_diag_admm_step_end_rows)
    cw, r2 = torch.empty_like(Wf), torch.empty_like(Wf)
    dev.diag_admm_cg_init(ops.c_mat.cpat, U, x0, ld, scale, rho, nlam, aval, r2, at=66, cw=cw)
    CUh = C @ Uh
    assert np.abs(cw.cpu().numpy() - CUh).max() <= 1e-12 * (1 + np.abs(CUh).max())
    ax2, lam2 = torch.empty_like(ax), torch.empty_like(ax)
    dev.diag_admm_step_end_rows(cw, U, V, ld, aval, ops.b, lam, rho, ax2, lam2, at=70)
    s2 = dev.fetch(73)
    assert np.abs(ax2.cpu().numpy() - axh).max() <= 1e-11 * (1 + np.abs(axh).max())
    assert np.abs(lam2.cpu().numpy() - ln).max() <= 1e-11 * (1 + np.abs(ln).max())
    assert close(s2[70], np.sum(CUh * Vh)) and close(s2[71], res @ res)
    assert close(s2[72], ln @ ops.b.cpu().numpy())


@pytest.mark.gpu
def test_step_end_rows_empty(dev):
    import torch
    e = torch.empty((0, 4), dtype=torch.float64, device="cuda")
    m = torch.empty(0, dtype=torch.float64, device="cuda")
    dev.slab[80:83] = 3.0
    dev.diag_admm_step_end_rows(e, e, e, 4, m, m, m, 1.0, m, m, at=80)
    assert list(dev.fetch(83)[80:83]) == [0.0, 0.0, 0.0]


@pytest.mark.parametrize("pq", [2.5, -1.0, 0.0, float("nan"), float("inf")])
def test_cg_step_dev_alpha_and_rejected_curvature(dev, pq):
    """cl_cg_step_dev: alpha = qr / pq on the device, bit-equal to the host division; a
    curvature cg_solve rejects (admm.py:83-86) leaves x and r untouched."""
    import ctypes
    import torch
    from paper_2407_15049_b200.device import ptr
    rng = np.random.default_rng(1)
    T = lambda: torch.as_tensor(rng.standard_normal((500, 6))).cuda().contiguous()  # noqa: E731
    x, p_, r, Q = T(), T(), T(), T()
    x0, r0 = x.clone(), r.clone()
    dev.slab[700] = pq
    qr = 3.7
    rc = dev.lib.cl_cg_step_dev(x.numel(), qr, dev.slot(700), ptr(x), ptr(x), ptr(p_), ptr(r), ptr(Q),
                                dev.slot(701), ptr(dev.ws), dev.sp)
    assert rc == 0
    torch.cuda.synchronize()
    if np.isfinite(pq) and pq > 0:
        alpha = qr / pq
        want_x = x0.cpu().numpy() + alpha * p_.cpu().numpy()
        want_r = r0.cpu().numpy() - alpha * Q.cpu().numpy()
        assert np.abs(x.cpu().numpy() - want_x).max() <= 1e-14 * (1 + np.abs(want_x).max())
        assert np.abs(r.cpu().numpy() - want_r).max() <= 1e-14 * (1 + np.abs(want_r).max())
        assert abs(dev.fetch(702)[701] - np.sum(want_r * want_r)) <= 1e-10 * np.sum(want_r * want_r)
    else:
        assert torch.equal(x, x0) and torch.equal(r, r0)
    del ctypes


@pytest.mark.gpu
@pytest.mark.parametrize("n,ld", [(0, 4), (1, 2), (777, 26), (4099, 64), (300, 202)])
def test_diag_cg_rows_pair_matches_stored_q(dev, n, ld):
    """cl_diag_cg_apply_rows + cl_diag_cg_step (Q rebuilt per row, never stored) give the
    same p, x and r bit for bit as cl_diag_cg_apply + cl_cg_step with a stored Q, and the
    same <p, Q>; host and device alpha agree."""
    import torch
    from paper_2407_15049_b200.device import ptr
    rng = np.random.default_rng(n + ld)
    T = lambda: torch.as_tensor(rng.standard_normal((n, ld))).cuda().contiguous()  # noqa: E731
    aval = torch.as_tensor(rng.standard_normal(n) + 2.0).cuda()
    Wf, p0, r0, x0 = T(), T(), T(), T()
    rho, beta = 1.7, 0.37
    if n == 0:            # empty problem: both calls succeed and report a zero dot
        coef = torch.empty(1, dtype=torch.float64, device="cuda")
        dev.slab[810:812] = 5.0
        dev.diag_cg_apply_rows(aval, ld, rho, p0, Wf, coef, r=r0, beta=beta, at=810)
        dev.diag_cg_step(ld, rho, coef, Wf, x0, x0, p0, r0, alpha=1.0, at=811)
        assert list(dev.fetch(812)[810:812]) == [0.0, 0.0]
        return
    # stored-Q reference
    p1, r1, x1, Q = p0.clone(), r0.clone(), x0.clone(), torch.empty_like(p0)
    dev.diag_cg_apply(aval, ld, rho, p1, Wf, Q, r=r1, beta=beta, at=800)
    pq = float(dev.fetch(801)[800])
    alpha = 2.3 / pq if n else 0.0
    dev.cg_step(alpha, x1, x1, p1, r1, Q, at=801)
    rr1 = float(dev.fetch(802)[801])
    # row-coefficient pair, host alpha then device alpha
    for dev_alpha in (False, True):
        p2, r2, x2 = p0.clone(), r0.clone(), x0.clone()
        coef = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
        dev.diag_cg_apply_rows(aval, ld, rho, p2, Wf, coef, r=r2, beta=beta, at=810)
        assert float(dev.fetch(811)[810]) == pq
        if dev_alpha and n:
            dev.diag_cg_step(ld, rho, coef, Wf, x2, x2, p2, r2, qr=2.3, pq_at=810, at=811)
        else:
            dev.diag_cg_step(ld, rho, coef, Wf, x2, x2, p2, r2, alpha=alpha, at=811)
        torch.cuda.synchronize()
        assert torch.equal(p1, p2) and torch.equal(x1, x2) and torch.equal(r1, r2)
        rr2 = float(dev.fetch(812)[811])
        assert abs(rr2 - rr1) <= 1e-12 * max(rr1, 1e-300)
    del ptr

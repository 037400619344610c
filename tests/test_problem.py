"""Host problem model and ingestion (CPU): same behaviour as lrsdp/problem.py."""

import io

import numpy as np
import pytest

from oracle import lrsdp_oracle as O
from paper_2407_15049_b200.exceptions import SdpaParseError, UnsupportedFeatureError
from paper_2407_15049_b200.problem import (GraphEdgeList, ObservationSet, SdpProblem,
                                           SymmetricSparse, build_matrix_completion, build_maxcut,
                                           parse_sdpa, read_edge_list, read_observations,
                                           serialize_sdpa, validate)
from tests._golden import load, ops_cases, problem_from

SMALLEST = "1\n1\n2\n1.0\n0 1 1 1 1.0\n1 1 1 1 1.0\n"


def triangle():
    return build_maxcut(GraphEdgeList.from_edges(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)]))


def rand_problem(rng, n, m):
    def sym(d):
        e = [(i, j, float(rng.standard_normal())) for i in range(n) for j in range(i, n)
             if rng.random() < d]
        return e or [(0, 0, 1.0)]
    con, row, col, val = [], [], [], []
    for k in range(m):
        for (i, j, v) in sym(0.3):
            con.append(k); row.append(i); col.append(j); val.append(v)
    return SdpProblem(n=n, m=m, C=SymmetricSparse.from_entries(n, sym(0.3)),
                      a_con=np.array(con, dtype=np.int64), a_row=np.array(row, dtype=np.int64),
                      a_col=np.array(col, dtype=np.int64), a_val=np.array(val), b=rng.standard_normal(m))


def test_smallest_sdpa_file_sign_convention():
    p = parse_sdpa(SMALLEST)
    assert (p.n, p.m, p.maximize) == (2, 1, True)
    assert p.C.to_dense()[0, 0] == -1.0 and p.C.to_dense()[0, 1] == 0.0
    assert p.constraint(0).to_dense()[0, 0] == 1.0 and p.b.tolist() == [1.0]


def test_sdpa_bytes_stream_comments_braces():
    ref = parse_sdpa(SMALLEST)
    assert parse_sdpa(SMALLEST.encode()) == ref
    assert parse_sdpa(io.StringIO(SMALLEST)) == ref
    assert parse_sdpa('"c\n* c\n1\n1\n{2}\n{1.0,}\n0 1 1 1 1.0\n1 1 1 1 1.0\n') == ref


@pytest.mark.parametrize("text,exc,msg", [
    ("1\n2\n2 2\n1.0\n0 1 1 1 1.0\n", UnsupportedFeatureError, None),
    ("1\n1\n-2\n1.0\n0 1 1 1 1.0\n", UnsupportedFeatureError, None),
    ("1\n1\n2\n1.0\n0 1 1 oops 1.0\n", SdpaParseError, "line 5"),
    ("1\n1\n2\n1.0\n0 1 3 3 1.0\n", SdpaParseError, None),
    ("1\n1\n2\n", SdpaParseError, "end of file"),
    ("1\n1\n2\n1.0\n0 2 1 1 1.0\n", UnsupportedFeatureError, None),
])
def test_sdpa_errors(text, exc, msg):
    with pytest.raises(exc, match=msg):
        parse_sdpa(text)


def test_sdpa_duplicates_summed_with_warning():
    with pytest.warns(UserWarning):
        p = parse_sdpa("1\n1\n2\n1.0\n1 1 1 2 1.0\n1 1 2 1 2.0\n")
    assert p.constraint(0).to_dense()[0, 1] == 3.0


def test_sdpa_roundtrip():
    rng = np.random.default_rng(1)
    for _ in range(20):
        p = rand_problem(rng, int(rng.integers(1, 9)), int(rng.integers(1, 6)))
        q = parse_sdpa(serialize_sdpa(p))
        assert parse_sdpa(serialize_sdpa(q)) == q


def test_lowrank_inner_and_norm1_match_dense():
    rng = np.random.default_rng(2)
    for _ in range(20):
        n = int(rng.integers(1, 12))
        C = rand_problem(rng, n, 1).C
        x = rng.standard_normal((n, 2))
        dense = float(np.sum(C.to_dense() * (x @ x.T)))
        assert abs(C.inner_lowrank(x, x) - dense) <= 1e-12 * (1 + abs(dense))
        assert np.isclose(C.vec_norm1(), np.abs(C.to_dense()).sum(), rtol=1e-13)


def test_maxcut_builders():
    p = triangle()
    L = np.array([[2., -1., -1.], [-1., 2., -1.], [-1., -1., 2.]])
    assert np.allclose(p.C.to_dense(), -L / 4.0) and p.m == 3 and np.all(p.b == 1.0)
    p1 = build_maxcut(GraphEdgeList.from_edges(2, [(0, 1, 3.0)]))
    assert np.allclose(p1.C.to_dense(), -np.array([[3., -3.], [-3., 3.]]) / 4.0)
    p0 = build_maxcut(GraphEdgeList.from_edges(1, []))
    assert p0.C.nnz_stored == 0 and p0.m == 1
    assert triangle().dense_c


def test_maxcut_builder_matches_golden_reference_output():
    z = load("ops_maxcut_g60.npz")
    p = problem_from(z)
    # rebuild from the graph encoded in the golden Laplacian
    off = z["c_rows"] != z["c_cols"]
    g = GraphEdgeList(int(z["n"]), z["c_rows"][off], z["c_cols"][off], 4.0 * z["c_vals"][off])
    q = build_maxcut(g)
    assert q == p


def test_completion_builder():
    p = build_matrix_completion(ObservationSet.from_triples(1, 1, [(0, 0, 5.0)]))
    A = p.constraint(0).to_dense()
    assert p.n == 2 and A[0, 1] == 1.0 and A[1, 0] == 1.0 and p.b.tolist() == [10.0]
    with pytest.raises(ValueError):
        build_matrix_completion(ObservationSet.from_triples(2, 2, []))


def test_validate_and_readers():
    d = validate(triangle())
    assert (d.nnz_a, d.nonzero_columns, d.index_ok, d.symmetry_ok) == (3, 3, True, True)
    p = parse_sdpa(SMALLEST)
    bad = SdpProblem(n=p.n, m=p.m, C=p.C, a_con=np.array([0]), a_row=np.array([1]),
                     a_col=np.array([0]), a_val=np.array([1.0]), b=p.b)
    assert not validate(bad).symmetry_ok
    g = read_edge_list("3\n1 2\n2 3 2.5\n")
    assert g.n == 3 and g.weights.tolist() == [1.0, 2.5]
    with pytest.raises(ValueError):
        read_edge_list("2\n1 1\n")
    with pytest.raises(ValueError):
        read_edge_list("3\n1 2\n2 1\n")
    o = read_observations("2 3\n1 1 0.5\n2 3 -1.0\n")
    assert (o.n2, o.n1) == (2, 3) and o.obs_val.tolist() == [0.5, -1.0]
    with pytest.raises(ValueError):
        read_observations("2 2\n1 1 1.0\n1 1 2.0\n")


@pytest.mark.parametrize("case", ops_cases())
def test_problem_norms_match_oracle(case):
    p = problem_from(load(f"ops_{case}.npz"))
    b1, binf, cn = O.norms(p)
    assert (p.b_norm1, p.b_norminf, p.c_vec_norm1) == (b1, binf, cn)
    assert p.nnz_a_full() == O.nnz_a_full(p)


def test_locality_permutation_is_a_relabelling():
    """reorder.permute: objective and constraint values invariant under the relabelling."""
    from paper_2407_15049_b200 import graphs, problem, reorder
    from oracle import lrsdp_oracle as O
    for p in (problem.build_maxcut(graphs.delaunay_like(400, seed=2)),
              problem.build_matrix_completion(graphs.random_completion(20, 15, 120, seed=2))):
        perm = reorder.locality_order(p)
        q, inv = reorder.permute(p, perm)
        assert np.array_equal(inv[perm], np.arange(p.n))
        rng = np.random.default_rng(0)
        U, V = rng.standard_normal((p.n, 3)), rng.standard_normal((p.n, 3))
        oa, ob = O.OracleOps(p), O.OracleOps(q)
        assert abs(oa.objective(U, V) - ob.objective(U[perm], V[perm])) <= 1e-10 * (1 + abs(oa.objective(U, V)))
        ax, bx = oa.A(U, V), ob.A(U[perm], V[perm])
        if reorder.is_diag(p):
            bx = bx[inv]
        assert np.abs(ax - bx).max() <= 1e-12 * (1 + np.abs(ax).max())
        assert reorder.is_diag(q) == reorder.is_diag(p)
    g = problem.build_maxcut(graphs.delaunay_like(900, seed=3))
    assert reorder.locality_gain(g, reorder.locality_order(g)) > 2.0

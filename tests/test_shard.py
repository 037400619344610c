"""Row-sharded solve plumbing on CPU: world_size 2 over gloo (shard.py).

The GPU kernels cannot run here, so the ghost-aware SpMM is emulated in
torch (``shard.local_spmm_reference``) on the remapped indices the kernels
consume; everything else -- block partition, publish lists, the all-gather
of boundary rows, halo positions, scalar all-reduce -- is the product code.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import scipy.sparse as sp
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(fn, world, *args):
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_entry, args=(world, port, fn, d, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, d, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, d, *args)
    finally:
        dist.destroy_process_group()


def _sym_pattern(n, seed, deg):
    rng = np.random.default_rng(seed)
    m = n * deg // 2
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    M = sp.coo_matrix((rng.standard_normal(m), (u, v)), shape=(n, n)).tocsr()
    M = (M + M.T + sp.diags(rng.standard_normal(n))).tocsr()
    M.sum_duplicates()
    M.sort_indices()
    return M


def _check_halo_spmm(rank, world, d, n, seed, deg, ld):
    from paper_2407_15049_b200 import shard
    M = _sym_pattern(n, seed, deg)
    X = np.random.default_rng(seed + 1).standard_normal((n, ld))
    b = shard.block_bounds(n, world)
    lo, hi = b[rank], b[rank + 1]
    rows = M[lo:hi]
    indptr = torch.as_tensor(rows.indptr.astype(np.int64))
    cols = torch.as_tensor(rows.indices.astype(np.int64))
    plan = shard.HaloPlan(lo, hi, indptr, cols, b, rank, world)
    Xl = torch.as_tensor(X[lo:hi]).contiguous()
    halo = plan.exchange(Xl, ld, shard.torch_pack)
    assert halo.shape == (world * plan.maxb, ld)
    got = shard.local_spmm_reference(indptr, plan.local_indices, torch.as_tensor(rows.data), Xl, halo,
                                     plan.nown)
    want = rows @ X
    assert np.abs(got.numpy() - want).max() <= 1e-12 * (1 + np.abs(want).max())
    # owned columns stay local, remote ones land past nown
    own = (cols >= lo) & (cols < hi)
    assert bool((plan.local_indices[own] < plan.nown).all())
    assert bool((plan.local_indices[~own] >= plan.nown).all())
    # every published row is referenced by some other rank (symmetry)
    assert plan.counts[rank] == plan.publish.numel()


@pytest.mark.parametrize("world,n,deg,ld", [(2, 300, 6, 4), (2, 1000, 10, 26), (3, 257, 4, 6)])
def test_halo_exchange_reproduces_global_spmm(world, n, deg, ld):
    _run(_check_halo_spmm, world, n, 7 + n, deg, ld)


def _check_block_diag(rank, world, d):
    """A block-diagonal pattern publishes nothing and needs no halo rows."""
    from paper_2407_15049_b200 import shard
    n = 100
    b = shard.block_bounds(n, world)
    lo, hi = b[rank], b[rank + 1]
    indptr = torch.arange(hi - lo + 1, dtype=torch.int64)
    cols = torch.arange(lo, hi, dtype=torch.int64)
    plan = shard.HaloPlan(lo, hi, indptr, cols, b, rank, world)
    assert plan.counts == [0] * world
    assert plan.publish.numel() == 0
    assert torch.equal(plan.local_indices.long(), torch.arange(hi - lo))


def test_block_diagonal_pattern_has_empty_halo():
    _run(_check_block_diag, 2)


def _check_maxcut_rows(rank, world, d):
    """Sharded Laplacian rows equal the single-process build_maxcut rows (problem.py:387)."""
    from paper_2407_15049_b200 import graphs, problem, shard
    n, deg = 500, 6.0
    eu, ev = shard.random_graph_edges(n, deg, 3, torch.device("cpu"))
    g = problem.GraphEdgeList(n, eu.numpy(), ev.numpy(), np.ones(eu.numel()))
    p = problem.build_maxcut(g)
    full = sp.csr_matrix((np.concatenate([p.C.vals, p.C.vals[p.C.rows != p.C.cols]]),
                          (np.concatenate([p.C.rows, p.C.cols[p.C.rows != p.C.cols]]),
                           np.concatenate([p.C.cols, p.C.rows[p.C.rows != p.C.cols]]))), shape=(n, n))
    b = shard.block_bounds(n, world)
    lo, hi = b[rank], b[rank + 1]
    indptr, cols, vals = shard.maxcut_rows(n, eu, ev, lo, hi)
    loc = sp.csr_matrix((vals.numpy(), cols.numpy(), indptr.numpy()), shape=(hi - lo, n))
    assert abs(loc - full[lo:hi]).max() == 0.0
    # the scalar all-reduce of a sharded dot product equals the global one
    X = np.random.default_rng(0).standard_normal((n, 4))
    part = torch.tensor([float(np.sum((loc @ X) * X[lo:hi]))], dtype=torch.float64)
    dist.all_reduce(part)
    want = float(np.sum((full @ X) * X))
    assert abs(part.item() - want) <= 1e-12 * (1 + abs(want))
    del graphs


def test_sharded_maxcut_rows_match_global_and_allreduce():
    _run(_check_maxcut_rows, 2)


def test_block_bounds_cover_rows():
    from paper_2407_15049_b200 import shard
    for n, w in [(10, 3), (7, 7), (1000, 8)]:
        b = shard.block_bounds(n, w)
        assert b[0] == 0 and b[-1] == n and all(b[k] <= b[k + 1] for k in range(w))


class _CpuDev:
    """The slice of device.Device the operator builders use (no kernels run)."""

    def __init__(self):
        self.dev = torch.device("cpu")

    def put(self, a, dtype=torch.float64):
        return torch.as_tensor(np.ascontiguousarray(a)).to(dtype=dtype)


def _same(a, b):
    if a is None or b is None:
        return a is None and b is None
    return a.dtype == b.dtype and torch.equal(a.cpu(), b.cpu())


def _check_local_diag_build(rank, world, d, n, deg):
    """The per-rank MaxCut build (no global operator build) equals slicing the global one."""
    from paper_2407_15049_b200 import graphs, problem, shard
    p = problem.build_maxcut(graphs.random_sparse(n, deg=deg, seed=5))
    dev = _CpuDev()
    a = shard.build_sharded_operators(p, rank, world, dev, None, local=False)
    b = shard.build_sharded_operators(p, rank, world, dev, None, local=True)
    for pa, pb in ((a.adj.omega, b.adj.omega), (a.adj.apat, b.adj.apat), (a.c_mat.cpat, b.c_mat.cpat)):
        for f in ("indptr", "indices", "cv", "at_ptr", "at_con", "at_val"):
            assert _same(getattr(pa, f), getattr(pb, f)), f
        assert pa.nrows == pb.nrows
        assert (pa.halo is None) == (pb.halo is None)
        if pa.halo is not None:
            assert pa.halo.counts == pb.halo.counts and torch.equal(pa.halo.publish, pb.halo.publish)
        assert pa.mhalo is None and pb.mhalo is None
    ca, cb = a.cop.con, b.cop.con
    for f in ("indptr", "colidx", "pi", "pj", "val", "diag_aval"):
        assert _same(getattr(ca, f), getattr(cb, f)), f
    assert ca.halo is None and cb.halo is None
    assert torch.equal(a.b, b.b) and torch.equal(a.diag_aval, b.diag_aval)
    assert a.omega_size_ref == b.omega_size_ref and a.cop.ncols == b.cop.ncols
    assert a.row_range == b.row_range and a.con_range == b.con_range
    assert a.problem.m == b.problem.m and a.problem.n == b.problem.n


@pytest.mark.parametrize("world,n,deg", [(2, 400, 6.0), (3, 301, 10.0)])
def test_local_diag_build_matches_global_slice(world, n, deg):
    _run(_check_local_diag_build, world, n, deg)


def test_streamed_row_block_draw_matches_global_draw():
    """A rank's block of the reference's global random draws (initial factor: divided by
    sqrt(n r0); escalation noise: multiplied by 1e-3/sqrt(n)) is bit-identical to slicing
    the full draw, and leaves the generator where the full draw leaves it."""
    import math
    from paper_2407_15049_b200 import driver
    old = driver._DRAW_CHUNK
    driver._DRAW_CHUNK = 7
    try:
        n, r = 50, 3
        full = np.random.default_rng(4).standard_normal((n, r)) / math.sqrt(n * r)
        full2 = np.random.default_rng(4).standard_normal((n, r)) * (1e-3 / math.sqrt(n))
        for lo, hi in [(0, 50), (3, 20), (13, 14), (49, 50)]:
            got = driver._draw(np.random.default_rng(4), n, r, rows=(lo, hi), div=math.sqrt(n * r))
            assert np.array_equal(got, full[lo:hi])
            got = driver._draw(np.random.default_rng(4), n, r, mult=1e-3 / math.sqrt(n), rows=(lo, hi))
            assert np.array_equal(got, full2[lo:hi])
        g1 = np.random.default_rng(4)
        driver._draw(g1, n, r, rows=(3, 9), div=2.0)
        g2 = np.random.default_rng(4)
        g2.standard_normal((n, r))
        assert np.array_equal(g1.standard_normal(5), g2.standard_normal(5))
    finally:
        driver._DRAW_CHUNK = old


def test_memory_model_configs():
    """DESIGN.md's per-rank memory table: configs[3] fits 8 ranks with room to escalate;
    configs[4] fits 8 ranks at its starting rank (a uniformly random graph only just:
    the all-gather halo is the whole remote factor, the peer halo about half of it)."""
    from paper_2407_15049_b200 import driver, shard
    budget = 0.94 * 183359 * 2 ** 20          # the driver's default: 94 % of a B200's 183359 MiB
    c3 = shard.memory_model(int(2e7), 8, 29, 0, m_global=int(2e8), nnz_a_per_con=2, halo_slots=2, pair=True)
    assert c3["total"] < budget / 4
    assert shard.memory_model(int(2e7), 8, 140, 0, m_global=int(2e8), nnz_a_per_con=2, halo_slots=2,
                              pair=True)["total"] < budget
    mesh = shard.memory_model(int(1.7e8), 8, 29, 7, halo_frac=0.002)
    rand = shard.memory_model(int(1.7e8), 8, 29, 7)
    peer = shard.memory_model(int(1.7e8), 8, 29, 7, peer=True)
    nv = shard.memory_model(int(1.7e8), 8, 29, 7, nvlink=True)
    assert nv["halo"] == 0 and nv["total"] == rand["total"] - rand["halo"]
    assert mesh["total"] < peer["total"] < rand["total"] < budget
    # the next rank (r0 = 29 -> 44) does not fit on any of them
    assert shard.memory_model(int(1.7e8), 8, 44, 7, halo_frac=0.002)["total"] > budget
    assert mesh["stage_buffers"] == driver.stage_factor_buffers(8) * mesh["factor_bytes"]
    # the driver's guard counts the same stage buffers
    assert driver.factor_bytes_needed(100, 100, 29, 8) >= driver.stage_factor_buffers(8) * 100 * 30 * 8


def _check_peer_halo_spmm(rank, world, d, n, seed, deg, ld):
    """The point-to-point halo (PeerHaloPlan) reproduces the global SpMM, receives only the
    referenced rows, and beats the all-gather on a random graph (make_halo_plan picks it)."""
    from paper_2407_15049_b200 import shard
    M = _sym_pattern(n, seed, deg)
    X = np.random.default_rng(seed + 1).standard_normal((n, ld))
    b = shard.block_bounds(n, world)
    lo, hi = b[rank], b[rank + 1]
    rows = M[lo:hi]
    indptr = torch.as_tensor(rows.indptr.astype(np.int64))
    cols = torch.as_tensor(rows.indices.astype(np.int64))
    plan = shard.PeerHaloPlan(lo, hi, indptr, cols, b, rank, world)
    Xl = torch.as_tensor(X[lo:hi]).contiguous()
    halo = plan.exchange(Xl, ld, shard.torch_pack)
    got = shard.local_spmm_reference(indptr, plan.local_indices, torch.as_tensor(rows.data), Xl,
                                     halo[:plan.halo_rows], plan.nown)
    want = rows @ X
    assert np.abs(got.numpy() - want).max() <= 1e-12 * (1 + np.abs(want).max())
    remote = np.unique(rows.indices[(rows.indices < lo) | (rows.indices >= hi)])
    assert plan.halo_rows == remote.size                       # exactly the referenced rows
    assert np.array_equal(halo[:plan.halo_rows].numpy(), X[remote])
    ag = shard.HaloPlan(lo, hi, indptr, cols, b, rank, world)
    auto = shard.make_halo_plan(lo, hi, indptr, cols, b, rank, world)
    assert max(plan.counts) < world * ag.maxb and isinstance(auto, shard.PeerHaloPlan)
    # the remap of any referenced column agrees with the local indices
    assert torch.equal(plan.remap(cols).to(torch.int32), plan.local_indices)


@pytest.mark.parametrize("world,n,deg,ld", [(2, 600, 6, 4), (3, 1000, 10, 26), (4, 257, 4, 6)])
def test_peer_halo_reproduces_global_spmm(world, n, deg, ld):
    _run(_check_peer_halo_spmm, world, n, 11 + n, deg, ld)


def _check_local_single_entry_build(rank, world, d, n2, n1, m):
    """The per-rank matrix-completion build (no global operator build) equals slicing the
    global one: patterns, halo plans, multiplier halo, renumbered constraint rows."""
    from paper_2407_15049_b200 import graphs, problem, shard
    p = problem.build_matrix_completion(graphs.random_completion(n2, n1, m, seed=7))
    assert shard.is_single_entry_problem(p) and not shard.is_diag_problem(p)
    dev = _CpuDev()
    a = shard.build_sharded_operators(p, rank, world, dev, None, local=False)
    b = shard.build_sharded_operators(p, rank, world, dev, None, local=True)
    for pa, pb in ((a.adj.omega, b.adj.omega), (a.adj.apat, b.adj.apat), (a.c_mat.cpat, b.c_mat.cpat)):
        for f in ("indptr", "indices", "cv", "at_ptr", "at_con", "at_val"):
            assert _same(getattr(pa, f), getattr(pb, f)), f
        assert pa.nrows == pb.nrows
        for h in ("halo", "mhalo"):
            ha, hb = getattr(pa, h), getattr(pb, h)
            assert (ha is None) == (hb is None), h
            if ha is not None:
                assert type(ha) is type(hb) and ha.counts == hb.counts and torch.equal(ha.publish, hb.publish)
    ca, cb = a.cop.con, b.cop.con
    for f in ("indptr", "pi", "pj", "val"):
        assert _same(getattr(ca, f), getattr(cb, f)), f
    assert (ca.halo is None) == (cb.halo is None)
    assert torch.equal(a.b, b.b) and a.diag_aval is None and b.diag_aval is None
    assert a.omega_size_ref == b.omega_size_ref and a.cop.ncols == b.cop.ncols
    assert a.row_range == b.row_range and a.con_range == b.con_range
    assert a.problem.m == b.problem.m and a.problem.n == b.problem.n


@pytest.mark.parametrize("world,n2,n1,m", [(2, 40, 30, 300), (3, 61, 47, 900)])
def test_local_single_entry_build_matches_global_slice(world, n2, n1, m):
    _run(_check_local_single_entry_build, world, n2, n1, m)


def _check_nvlink_plan(rank, world, d, n, seed, deg, ld):
    """Peer-memory plan (shard.NvlinkHaloPlan): remote columns are encoded as
    CL_PEER_COL(owner, row), decode to the global ids, and a product that reads each
    encoded row from its owner's block (what the GHOST 2 SpMM does over NVLink) equals the
    global product. No halo buffer, no collective on the data path."""
    from paper_2407_15049_b200 import shard
    M = _sym_pattern(n, seed, deg)
    X = np.random.default_rng(seed + 1).standard_normal((n, ld))
    b = shard.block_bounds(n, world)
    lo, hi = b[rank], b[rank + 1]
    rows = M[lo:hi]
    indptr = torch.as_tensor(rows.indptr.astype(np.int64))
    cols = torch.as_tensor(rows.indices.astype(np.int64))
    plan = shard.make_halo_plan(lo, hi, indptr, cols, b, rank, world, mode="nvlink", peer_ok=True)
    assert isinstance(plan, shard.NvlinkHaloPlan) and plan.ghost_nown == shard.GHOST_PEERS
    # without peer_ok (patterns other kernels read too) the copy-based plans are used
    assert not isinstance(shard.make_halo_plan(lo, hi, indptr, cols, b, rank, world, mode="nvlink"),
                          shard.NvlinkHaloPlan)
    li = plan.local_indices.to(torch.int64)
    own = (cols >= lo) & (cols < hi)
    assert plan.local_indices.dtype == torch.int32
    assert bool((li[own] >= 0).all()) and bool((li[~own] < 0).all())
    assert torch.equal(shard.decode_peer_columns(li, lo, b), cols)
    assert plan.counts[rank] == int((~own).sum()) and sum(plan.counts) > 0
    assert plan.halo_rows == 0 and plan.maxb == 0 and plan.halo_bytes(ld) == int((~own).sum()) * ld * 8
    # emulate the kernel: owner = bits 28..30, row = bits 0..27 of the unsigned index
    blocks = [torch.as_tensor(X[b[k]:b[k + 1]]) for k in range(world)]
    u = li + (1 << 31)
    got = torch.zeros((hi - lo, ld), dtype=torch.float64)
    vals = torch.as_tensor(rows.data)
    for i in range(hi - lo):
        for s in range(int(indptr[i]), int(indptr[i + 1])):
            j = int(li[s])
            src = blocks[rank][j] if j >= 0 else blocks[int(u[s]) >> 28 & 7][int(u[s]) & ((1 << 28) - 1)]
            got[i] += vals[s] * src
    want = rows @ X
    assert np.abs(got.numpy() - want).max() <= 1e-12 * (1 + np.abs(want).max())


@pytest.mark.parametrize("world,n,deg,ld", [(2, 300, 6, 4), (3, 401, 8, 6)])
def test_nvlink_plan_encodes_remote_rows(world, n, deg, ld):
    _run(_check_nvlink_plan, world, n, 5 + n, deg, ld)


def test_peer_column_encoding_limits():
    from paper_2407_15049_b200 import shard
    owner = torch.tensor([0, 1, 7, 7])
    row = torch.tensor([0, 5, (1 << 28) - 1, 3])
    enc = shard.peer_cols(owner, row)
    assert bool((enc < 0).all()) and bool((enc >= -(1 << 31)).all())
    assert torch.equal(enc.to(torch.int32).to(torch.int64), enc)        # fits the int32 index
    bounds = [0, 10, 20, 30, 40, 50, 60, 70, 1 << 29]
    dec = shard.decode_peer_columns(enc, 5, bounds)
    assert dec.tolist() == [0 + 0, 10 + 5, 70 + (1 << 28) - 1, 70 + 3]
    with pytest.raises(ValueError):
        shard.NvlinkHaloPlan(0, 1, torch.zeros(2, dtype=torch.int64), torch.zeros(1, dtype=torch.int64),
                             [0, 1, 2 ** 28 + 2], 0, 2)

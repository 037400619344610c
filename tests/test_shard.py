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

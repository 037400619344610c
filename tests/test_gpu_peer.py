"""Peer-memory ghost rows (shard.NvlinkHaloPlan, include/culorads.h CL_GHOST_PEERS).

The SpMM reads each remote factor row in place from its owner's memory: a pattern
column encoded as CL_PEER_COL(owner, row) loads ``table[owner] + row * ld``. On the one
GPU of the test box the "peers" are separate allocations on cuda:0 (the kernel cannot
tell a local address from an NVLink-mapped one), so every kernel variant that reads ghost
rows -- plain store, fused epilogue with dots, heavy rows, the diagonal-ADMM start and
step end -- is checked here against the same rows with global column indices on the
whole factor: the slot order and the loaded values are the same, so the results are
bit-identical. The IPC mapping itself and the fences are exercised by the two-process
solve at the bottom (two ranks sharing cuda:0 over gloo).
"""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch

pytestmark = pytest.mark.gpu


class _LocalPeers:
    """A stand-in NvlinkHaloPlan whose 'peers' are this process's row blocks of X."""

    ghost_nown = -2
    nown = 0

    def __init__(self, bounds, ld_blocks):
        self.bounds = bounds
        self.blocks = ld_blocks        # callable X -> list of per-rank block tensors
        self.released = 0

    def exchange(self, X, ld, pack=None, slot=0):
        from paper_2407_15049_b200 import shard
        tab = (shard.ctypes.c_uint64 * shard.MAX_PEERS)()
        for k, blk in enumerate(self.blocks(X)):
            tab[k] = blk.data_ptr()
        self._tab = tab                # the launch reads the table after exchange returns
        return shard._HostTable(tab)

    def release(self, X):
        self.released += 1


def _pattern(n, seed, deg, heavy=()):
    rng = np.random.default_rng(seed)
    m = n * deg // 2
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    for h in heavy:                      # dense rows: the kernel's global (heavy-tile) path
        u = np.concatenate([u, np.full(n // 2, h)])
        v = np.concatenate([v, rng.choice(n, n // 2, replace=False)])
    M = sp.coo_matrix((rng.standard_normal(len(u)), (u, v)), shape=(n, n)).tocsr()
    M = (M + M.T + sp.diags(rng.standard_normal(n))).tocsr()
    M.sum_duplicates()
    M.sort_indices()
    return M


def _dev_pattern(rows, indices):
    from paper_2407_15049_b200.linops import DevicePattern, padded
    ptr = torch.zeros(rows.shape[0] + 1 + 16, dtype=torch.int64, device="cuda")
    ptr[:rows.shape[0] + 1] = torch.as_tensor(rows.indptr.astype(np.int64))
    return DevicePattern(rows.shape[0], ptr[:rows.shape[0] + 1], padded(indices.to(torch.int32).cuda()),
                         padded(torch.as_tensor(rows.data).cuda()), None, None, None)


class _LocalHalo:
    """The copy-halo layout (HaloPlan-like): remote column t-th distinct id -> nown + t."""

    def __init__(self, nown, halo):
        self.nown = self.ghost_nown = nown
        self.halo = halo

    def exchange(self, X, ld, pack=None, slot=0):
        return self.halo


def _halo_ref(rows, cols, lo, hi, Wg):
    """Pattern + stub plan of the halo-buffer path (GHOST 1) for rows [lo, hi)."""
    own = (cols >= lo) & (cols < hi)
    rem = torch.unique(cols[~own])
    loc = cols - lo
    loc[~own] = (hi - lo) + torch.searchsorted(rem, cols[~own])
    pat = _dev_pattern(rows, loc)
    pat.halo = _LocalHalo(hi - lo, Wg[rem.cuda()].contiguous())
    return pat


def _blocks_of(Xs, ld):
    return lambda X: Xs


@pytest.mark.parametrize("n,deg,ld,world,heavy", [(3000, 8, 26, 3, ()), (2000, 6, 1, 2, ()),
                                                  (2500, 10, 64, 4, (17, 1800)), (1200, 6, 8, 8, (5,))])
def test_peer_ghost_spmm_bit_identical(n, deg, ld, world, heavy):
    from paper_2407_15049_b200 import shard
    from paper_2407_15049_b200.device import Device
    torch.cuda.set_device(0)
    dev = Device()
    M = _pattern(n, 7 + n, deg, heavy)
    b = shard.block_bounds(n, world)
    rng = np.random.default_rng(3)
    Xg = torch.as_tensor(rng.standard_normal((n, ld))).cuda()
    Yg = torch.as_tensor(rng.standard_normal((n, ld))).cuda()
    # every rank's block in its own allocation (what the peers' factors are)
    Xs = [Xg[b[k]:b[k + 1]].clone() for k in range(world)]
    for rank in range(world):
        lo, hi = b[rank], b[rank + 1]
        rows = M[lo:hi]
        cols = torch.as_tensor(rows.indices.astype(np.int64))
        enc = shard.encode_peer_columns(cols, lo, hi, b)
        assert bool((enc < 0).any()) or world == 1
        peer = _dev_pattern(rows, enc)
        peer.halo = _LocalPeers(b, _blocks_of(Xs, ld))
        ref = _dev_pattern(rows, cols)                # global columns on the whole factor
        Xl = Xs[rank]
        Yl = Yg[lo:hi].contiguous()
        # plain store (EPI 0)
        o1 = torch.empty((hi - lo, ld), dtype=torch.float64, device="cuda")
        o2 = torch.empty_like(o1)
        dev.spmm(peer, Xl, ld, alpha=0.5, out=o1, c_coeff=1.0)
        dev.spmm(ref, Xg, ld, alpha=0.5, out=o2, c_coeff=1.0)
        assert torch.equal(o1, o2), (rank, float((o1 - o2).abs().max()))
        want = 0.5 * (rows @ Xg.cpu().numpy())
        assert np.abs(o1.cpu().numpy() - want).max() <= 1e-12 * (1 + np.abs(want).max())
        # fused epilogue: out = S X + 2 Y, dots <out, Y>, <out, out>
        dev.spmm(peer, Xl, ld, out=o1, Y=(Yl,), ycoef=(2.0,), dots=[("out", ("y", 0)), ("out", "out")], at=0,
                 c_coeff=1.0)
        d1 = dev.fetch(2).copy()
        dev.spmm(ref, Xg, ld, out=o2, Y=(Yl,), ycoef=(2.0,), dots=[("out", ("y", 0)), ("out", "out")], at=0,
                 c_coeff=1.0)
        d2 = dev.fetch(2).copy()
        assert torch.equal(o1, o2) and np.array_equal(d1, d2), rank
        assert peer.halo.released == 2


@pytest.mark.parametrize("ld,world", [(26, 3), (8, 2)])
def test_peer_ghost_diag_admm_bit_identical(ld, world):
    """cl_diag_admm_cg_init (EPI 2) and cl_diag_admm_step_end (EPI 3) with peer ghosts, against
    the halo-buffer ghosts (the epilogues read local rows of the same operands)."""
    from paper_2407_15049_b200 import shard
    from paper_2407_15049_b200.device import Device
    torch.cuda.set_device(0)
    dev = Device()
    n = 4000
    M = _pattern(n, 11, 6)
    b = shard.block_bounds(n, world)
    rng = np.random.default_rng(9)
    Wg = torch.as_tensor(rng.standard_normal((n, ld))).cuda()
    Ws = [Wg[b[k]:b[k + 1]].clone() for k in range(world)]
    for rank in range(world):
        lo, hi = b[rank], b[rank + 1]
        nl = hi - lo
        rows = M[lo:hi]
        cols = torch.as_tensor(rows.indices.astype(np.int64))
        peer = _dev_pattern(rows, shard.encode_peer_columns(cols, lo, hi, b))
        peer.halo = _LocalPeers(b, _blocks_of(Ws, ld))
        ref = _halo_ref(rows, cols, lo, hi, Wg)       # the halo-buffer path on the same local operands
        x0 = torch.as_tensor(rng.standard_normal((nl, ld))).cuda()
        nlam = torch.as_tensor(rng.standard_normal(nl)).cuda()
        aval = torch.ones(nl, dtype=torch.float64, device="cuda")
        bv = torch.ones(nl, dtype=torch.float64, device="cuda")
        outs = []
        for pat, W in ((peer, Ws[rank]), (ref, Ws[rank])):
            r = torch.empty((nl, ld), dtype=torch.float64, device="cuda")
            cw = torch.empty_like(r)
            dev.diag_admm_cg_init(pat, W, x0, ld, 0.7, 3.0, nlam, aval, r, 0, cw=cw)
            s1 = dev.fetch(2).copy()
            ax = torch.empty(nl, dtype=torch.float64, device="cuda")
            ln = torch.empty_like(ax)
            dev.diag_admm_step_end(pat, x0, W, ld, aval, bv, nlam, 3.0, ax, ln, 0)
            s2 = dev.fetch(3).copy()
            outs.append((r, cw, s1, ax, ln, s2))
        (r1, c1, a1, x1, l1, b1), (r2, c2, a2, x2, l2, b2) = outs
        assert torch.equal(r1, r2) and torch.equal(c1, c2) and np.array_equal(a1, a2), rank
        assert torch.equal(x1, x2) and torch.equal(l1, l2) and np.array_equal(b1, b2), rank
        assert peer.halo.released == 2


def test_peer_ghosts_rejected_by_constraint_kernels():
    """Only the SpMM reads peer-encoded columns: the constraint kernels refuse the mode."""
    import ctypes

    from paper_2407_15049_b200 import _lib
    lib = _lib.load()
    t = torch.zeros(64, dtype=torch.float64, device="cuda")
    ip = torch.zeros(18, dtype=torch.int64, device="cuda")
    ip[1] = 1
    ix = torch.zeros(16, dtype=torch.int32, device="cuda")
    p = ctypes.c_void_p
    garr = (ctypes.c_void_p * 6)(*[t.data_ptr()] * 6)
    rc = lib.cl_constraint_eval_halo(1, p(ip.data_ptr()), p(ix.data_ptr()), p(ix.data_ptr()), p(t.data_ptr()), 2,
                                     p(t.data_ptr()), p(t.data_ptr()), None, None, p(t.data_ptr()), None, None,
                                     None, garr, _lib.CL_GHOST_PEERS, None)
    assert rc == _lib.CL_EARG


def test_ipc_export_reports_allocation_offset():
    import ctypes

    from paper_2407_15049_b200 import _lib
    lib = _lib.load()
    t = torch.zeros(1 << 20, dtype=torch.float64, device="cuda")
    h1 = (ctypes.c_uint8 * _lib.CL_IPC_HANDLE_BYTES)()
    h2 = (ctypes.c_uint8 * _lib.CL_IPC_HANDLE_BYTES)()
    o1, o2 = ctypes.c_int64(-1), ctypes.c_int64(-1)
    assert lib.cl_ipc_export(ctypes.c_void_p(t.data_ptr()), h1, ctypes.byref(o1)) == 0
    assert lib.cl_ipc_export(ctypes.c_void_p(t.data_ptr() + 8 * 1000), h2, ctypes.byref(o2)) == 0
    assert bytes(h1) == bytes(h2) and o2.value - o1.value == 8000 and o1.value >= 0


# ---------------------------------------------------------------------------
# two ranks on cuda:0: IPC-mapped peers, fences, the native loops' release hook
# ---------------------------------------------------------------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _peer_solve_worker(rank, world, port, case, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2407_15049_b200 import driver, shard
        from paper_2407_15049_b200.device import Device
        from tests._golden import cfg_of, load, problem_from
        z = load(f"solve_{case}.npz")
        p = problem_from(z)
        out = []
        for mode in ("nvlink", "allgather"):
            shard.HALO_MODE = mode
            rep = shard.solve_sharded(p, driver.SolverConfig(**dict(cfg_of(z))), dev=Device())
            out.append((mode, np.array([r[2:7] for r in rep.trace_rows], dtype=float), rep.objective,
                        rep.status, rep.gpu_launches))
        q.put((rank, out))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("g1_like", 2), ("maxcut_2k_deg6", 3)])
def test_peer_memory_sharded_solve_matches_halo_solve(case, world):
    """A row-sharded solve whose C products read remote rows in place from the other ranks'
    memory (CUDA IPC, stream fences; native ALM/ADMM loops with the release hook) gives the
    bit-identical trace and objective of the all-gather halo solve."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pc = mp.spawn(_peer_solve_worker, args=(world, _free_port(), case, q), nprocs=world, join=False)
    res = [q.get(timeout=900) for _ in range(world)]
    while not pc.join():
        pass
    for rank, out in res:
        assert not isinstance(out, str), out
        (m1, t1, o1, s1, l1), (m2, t2, o2, s2, l2) = out
        print(f"{case} rank {rank}: rows {len(t1)} objective {o1!r} status {s1} launches {l1} / {l2}")
        assert len(t1) == len(t2) and np.array_equal(t1, t2) and o1 == o2 and s1 == s2

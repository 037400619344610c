"""Peer-memory ghost rows (shard.NvlinkHaloPlan, include/culorads.h CL_GHOST_PEERS).

The SpMM reads each remote factor row in place from its owner's memory: a pattern
column encoded as CL_PEER_COL(owner, row) loads ``table[owner] + row * ld``. On the one
GPU of the test box the "peers" are separate allocations on cuda:0 (the kernel cannot
tell a local address from an NVLink-mapped one), so every kernel variant that reads ghost
rows -- plain store, fused epilogue with dots, heavy rows, the diagonal-ADMM start and
step end -- is checked here against the same rows with global column indices on the
whole factor: the slot order and the loaded values are the same, so the results are
bit-identical. The constraint kernel (matrix completion's A(UV^T) and the line search's three
products) reads its positions' remote rows the same way. The IPC mapping itself and the
fences are exercised by the two-process solves at the bottom (ranks sharing cuda:0 over
gloo).
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


class _OperandPeers(_LocalPeers):
    """Peer tables per operand: each local operand maps to its global blocks."""

    def __init__(self, table):
        self.table = table             # id(local operand) -> list of per-rank blocks
        self.released = 0
        self._tabs = []

    def exchange(self, X, ld, pack=None, slot=0):
        from paper_2407_15049_b200 import shard
        tab = (shard.ctypes.c_uint64 * shard.MAX_PEERS)()
        for k, blk in enumerate(self.table[id(X)]):
            tab[k] = blk.data_ptr()
        self._tabs.append(tab)
        return shard._HostTable(tab)


@pytest.mark.parametrize("world,ld", [(3, 26), (2, 8), (4, 2)])
def test_peer_ghost_constraint_kernel_bit_identical(world, ld):
    """cl_constraint_eval_halo in the peer mode (single-entry style constraints whose
    positions reference any rank's rows): one and three products, against the same
    constraint rows with global positions on whole factors."""
    from paper_2407_15049_b200 import shard
    from paper_2407_15049_b200.device import Device
    from paper_2407_15049_b200.linops import ConstraintCSR, padded
    torch.cuda.set_device(0)
    dev = Device()
    n, m = 3000, 5000
    rng = np.random.default_rng(21 + world)
    b = shard.block_bounds(n, world)
    lens = rng.integers(1, 3, m)
    ptr = np.concatenate([[0], np.cumsum(lens)])
    pi = rng.integers(0, n, ptr[-1])
    pj = rng.integers(0, n, ptr[-1])
    val = rng.standard_normal(ptr[-1])
    G = {k: torch.as_tensor(rng.standard_normal((n, ld))).cuda() for k in "UVD"}
    blocks = {k: [G[k][b[q]:b[q + 1]].clone() for q in range(world)] for k in "UVD"}
    bm = shard.block_bounds(m, world)
    for rank in range(world):
        lo, hi = b[rank], b[rank + 1]
        c0, c1 = bm[rank], bm[rank + 1]
        s0, s1 = ptr[c0], ptr[c1]
        T = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dt)   # noqa: E731
        cptr = torch.zeros(c1 - c0 + 1 + 16, dtype=torch.int64, device="cuda")
        cptr[:c1 - c0 + 1] = T(ptr[c0:c1 + 1] - s0, torch.int64)

        def con_of(pi_, pj_):
            return ConstraintCSR(m=c1 - c0, indptr=cptr[:c1 - c0 + 1], colidx=padded(T(np.zeros(s1 - s0), torch.int32)),
                                 pi=padded(pi_.to(torch.int32)), pj=padded(pj_.to(torch.int32)),
                                 val=padded(T(val[s0:s1], torch.float64)), diag_aval=None)
        gpi, gpj = T(pi[s0:s1], torch.int64), T(pj[s0:s1], torch.int64)
        peer = con_of(shard.encode_peer_columns(gpi, lo, hi, b), shard.encode_peer_columns(gpj, lo, hi, b))
        U, V, D = (blocks[k][rank] for k in "UVD")
        peer.halo = _OperandPeers({id(U): blocks["U"], id(V): blocks["V"], id(D): blocks["D"]})
        ref = con_of(gpi, gpj)
        o = [torch.empty(c1 - c0, dtype=torch.float64, device="cuda") for _ in range(6)]
        dev.constraint_eval(peer, ld, U, V, o[0])
        dev.constraint_eval(ref, ld, G["U"], G["V"], o[1])
        dev.constraint_eval(peer, ld, U, V, o[2], X2=V, Y2=U, X3=D, Y3=D, out2=o[3])
        dev.constraint_eval(ref, ld, G["U"], G["V"], o[4], X2=G["V"], Y2=G["U"], X3=G["D"], Y3=G["D"], out2=o[5])
        torch.cuda.synchronize()
        assert torch.equal(o[0], o[1]) and torch.equal(o[2], o[4]) and torch.equal(o[3], o[5]), rank
        Ug, Vg, Dg = (G[k].cpu().numpy() for k in "UVD")
        want = np.array([sum(val[t] * Ug[pi[t]] @ Vg[pj[t]] for t in range(ptr[c], ptr[c + 1]))
                         for c in range(c0, c1)])
        assert np.abs(o[0].cpu().numpy() - want).max() <= 1e-12 * (1 + np.abs(want).max())
        assert peer.halo.released == 2


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


def _peer_solve_worker(rank, world, port, case, q, over=None):
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
            cfg = dict(cfg_of(z))
            cfg.update(over or {})
            rep = shard.solve_sharded(p, driver.SolverConfig(**cfg), dev=Device())
            out.append((mode, np.array([r[2:7] for r in rep.trace_rows], dtype=float), rep.objective,
                        rep.status, rep.gpu_launches))
        q.put((rank, out))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("g1_like", 2), ("maxcut_2k_deg6", 3), ("completion_30", 2),
                                        ("completion_30", 3)])
def test_peer_memory_sharded_solve_matches_halo_solve(case, world):
    """A row-sharded solve whose C products (and, for matrix completion, constraint
    evaluations and Omega products) read remote rows in place from the other ranks' memory
    (CUDA IPC, stream fences; MaxCut's native ALM/ADMM loops with the release hook) gives
    the bit-identical trace and objective of the all-gather halo solve."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    # matrix completion (constraint rows and Omega through the peer plan): a capped solve,
    # the gloo-staged multiplier halo is slow
    over = dict(admm_step_cap=40, max_reopts=0) if case.startswith("completion") else None
    pc = mp.spawn(_peer_solve_worker, args=(world, _free_port(), case, q, over), nprocs=world, join=False)
    res = [q.get(timeout=900) for _ in range(world)]
    while not pc.join():
        pass
    for rank, out in res:
        assert not isinstance(out, str), out
        (m1, t1, o1, s1, l1), (m2, t2, o2, s2, l2) = out
        print(f"{case} rank {rank}: rows {len(t1)} objective {o1!r} status {s1} launches {l1} / {l2}")
        assert len(t1) == len(t2) and np.array_equal(t1, t2) and o1 == o2 and s1 == s2

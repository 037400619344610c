"""Row-sharded operators for the multi-GPU solve (north_star: "the n rows of the
factors and the matching CSR row blocks shard across the GPUs; remote factor
rows come in by all-gather or halo exchange; scalars combine by all-reduce").

Layout on rank k of P (one process per GPU, ``torch.distributed``):

* rows [lo_k, hi_k) of every n x ld factor, stored as a local nown x ld
  array (nown = hi_k - lo_k); m-vectors of row-aligned constraints likewise;
* the pattern rows of that block, column indices remapped to
  ``[0, nown)`` for owned columns and ``nown + r*maxb + t`` for the t-th
  published row of rank r -- the position that row lands at in the halo
  buffer after the all-gather;
* a halo buffer of P*maxb rows (``maxb`` = largest published set): before a
  product, each rank packs the rows other ranks reference (its *boundary*
  rows, a gather kernel) and all-gathers them. The SpMM kernel reads column
  j < nown from the local factor and j >= nown from the halo buffer
  (``cl_pattern.ghost``).

Patterns are symmetric (C and Omega are), so a row is referenced by another
rank exactly when it has a column in that rank's block: every rank derives
its own publish list locally, and one all-gather of the lists at setup
gives every rank the halo positions of the remote columns it references.

Every reduction of the solve is a sum over rows (or row-aligned
constraints), so the scalar slab is all-reduced (SUM) before the host reads
it and every rank takes the same algorithmic decision.

The plan is backend-agnostic (CPU tensors + gloo in the tests, CUDA tensors
+ NCCL on the GPU); packing is a callback so the tests can emulate the
gather kernel.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

I32 = torch.int32
I64 = torch.int64


def block_bounds(n, world):
    """Contiguous row blocks: rank k owns [b[k], b[k+1])."""
    return [k * n // world for k in range(world + 1)]


def _nccl(group=None):
    return dist.get_backend(group) == "nccl"


def _all_gather_1d(t, world, group=None):
    """All-gather equal-length 1-D tensors -> (world, len) tensor (works on gloo and NCCL)."""
    if world == 1:
        return t.view(1, -1)
    if t.is_cuda and _nccl(group):
        out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out.view(world, -1)
    # gloo (CPU tests, or several ranks sharing one GPU): stage through host memory
    h = t.detach().cpu().contiguous()
    parts = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(parts, h, group=group)
    return torch.stack(parts).to(t.device)


def all_reduce_sum(t, group=None):
    """In-place SUM all-reduce that also works for CUDA tensors on gloo."""
    if t.is_cuda and not _nccl(group):
        h = t.detach().cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)
    return t


class HaloPlan:
    """Publish/receive plan of one row-sharded symmetric pattern.

    ``indptr`` (nown+1) and ``indices`` (global column ids) are the local CSR
    rows [lo, hi) of a pattern; after construction ``local_indices`` holds
    the remapped int32 column indices the kernels use.
    """

    def __init__(self, lo, hi, indptr, indices, bounds, rank, world, group=None):
        self.lo, self.hi, self.rank, self.world, self.group = lo, hi, rank, world, group
        self.nown = nown = hi - lo
        dev = indices.device
        indices = indices.to(I64)
        counts_row = (indptr[1:] - indptr[:-1]).to(I64)
        rows = torch.repeat_interleave(torch.arange(nown, device=dev, dtype=I64), counts_row)
        own = (indices >= lo) & (indices < hi)
        publish = torch.unique(rows[~own])                      # sorted local row ids
        nb = torch.tensor([publish.numel()], dtype=I64, device=dev)
        counts = _all_gather_1d(nb, world, group).view(-1)
        self.counts = counts.cpu().tolist()
        self.maxb = maxb = max(1, max(self.counts))
        padded = torch.full((maxb,), -1, dtype=I64, device=dev)
        padded[:publish.numel()] = publish + lo
        lists = _all_gather_1d(padded, world, group)             # (world, maxb) global ids, -1 padded
        self.publish = publish.to(I32).contiguous()             # local rows this rank sends

        remote = indices[~own]
        bt = torch.tensor(bounds, dtype=I64, device=dev)
        owner = torch.searchsorted(bt, remote, right=True) - 1
        big = torch.iinfo(I64).max
        keyed = torch.where(lists >= 0, lists, torch.full_like(lists, big))
        # position of each remote column inside its owner's (sorted) publish list
        pos = torch.empty_like(remote)
        for r in range(world):
            sel = owner == r
            if bool(sel.any()):
                pos[sel] = torch.searchsorted(keyed[r].contiguous(), remote[sel])
        if remote.numel():
            found = lists[owner, pos.clamp(max=maxb - 1)]
            if not bool((found == remote).all()):
                raise ValueError("pattern is not symmetric across the row blocks: a referenced "
                                 "remote row is missing from its owner's publish list")
        loc = indices - lo
        loc[~own] = nown + owner * maxb + pos
        if nown + world * maxb >= 2 ** 31:
            raise ValueError("row block plus halo exceeds int32 column indices")
        self.local_indices = loc.to(I32).contiguous()
        self.halo_rows = world * maxb
        self._bufs = {}

    def buffers(self, ld, like):
        key = (ld, like.device)
        b = self._bufs.get(key)
        if b is None:
            send = torch.zeros((self.maxb, ld), dtype=like.dtype, device=like.device)
            recv = torch.zeros((self.world * self.maxb, ld), dtype=like.dtype, device=like.device)
            b = self._bufs[key] = (send, recv)
        return b

    def exchange(self, X, ld, pack):
        """Pack this rank's published rows of X and all-gather them; returns the halo buffer."""
        send, recv = self.buffers(ld, X)
        pack(self.publish, X.reshape(-1, ld), send)
        if self.world == 1:
            recv.copy_(send)
        elif recv.is_cuda and _nccl(self.group):
            dist.all_gather_into_tensor(recv, send, group=self.group)
        else:
            h = send.cpu()
            parts = [torch.empty_like(h) for _ in range(self.world)]
            dist.all_gather(parts, h, group=self.group)
            recv.view(self.world, self.maxb, ld).copy_(torch.stack(parts))
        return recv

    def halo_bytes(self, ld):
        """Bytes this rank receives per exchange (NVLink traffic of one halo)."""
        return (self.world - 1) * self.maxb * ld * 8


def torch_pack(idx, X, out):
    """Reference packing (tests): out[i] = X[idx[i]]."""
    out[:idx.numel()] = X[idx.long()]


def local_spmm_reference(indptr, local_indices, vals, X_local, halo, nown):
    """Dense emulation of the ghost-aware SpMM (tests): rows of S @ [X_local; halo]."""
    ext = torch.cat([X_local, halo], 0)
    nrows = indptr.numel() - 1
    out = torch.zeros((nrows, X_local.shape[1]), dtype=X_local.dtype)
    for i in range(nrows):
        a, b = int(indptr[i]), int(indptr[i + 1])
        if b > a:
            out[i] = (vals[a:b, None] * ext[local_indices[a:b].long()]).sum(0)
    return out


# ---------------------------------------------------------------------------
# row-sharded MaxCut operators (bench.py --gpus N, weak scaling)
# ---------------------------------------------------------------------------

def random_graph_edges(n, deg, seed, device):
    """The same seeded random simple graph on every rank (u < v, unit weights)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    me = int(round(n * deg / 2))
    u = torch.randint(0, n, (me,), generator=g, device=device, dtype=I64)
    v = torch.randint(0, n, (me,), generator=g, device=device, dtype=I64)
    a, b = torch.minimum(u, v), torch.maximum(u, v)
    keep = a != b
    code = torch.unique(a[keep] * n + b[keep])
    return code // n, code % n


def maxcut_rows(n, eu, ev, lo, hi):
    """Rows [lo, hi) of C = -L/4 (problem.py:387 build_maxcut): CSR with global columns."""
    dev = eu.device
    nown = hi - lo
    deg = torch.zeros(nown, dtype=torch.float64, device=dev)
    for x in (eu, ev):
        sel = (x >= lo) & (x < hi)
        deg.index_add_(0, x[sel] - lo, torch.ones(int(sel.sum()), dtype=torch.float64, device=dev))
    s1 = (eu >= lo) & (eu < hi)
    s2 = (ev >= lo) & (ev < hi)
    rows = torch.cat([torch.arange(lo, hi, device=dev, dtype=I64), eu[s1], ev[s2]])
    cols = torch.cat([torch.arange(lo, hi, device=dev, dtype=I64), ev[s1], eu[s2]])
    vals = torch.cat([-0.25 * deg, torch.full((int(s1.sum()) + int(s2.sum()),), 0.25,
                                              dtype=torch.float64, device=dev)])
    order = torch.argsort((rows - lo) * n + cols)
    rows, cols, vals = rows[order], cols[order], vals[order]
    indptr = torch.zeros(nown + 1, dtype=I64, device=dev)
    indptr[1:] = torch.cumsum(torch.bincount(rows - lo, minlength=nown), 0)
    return indptr, cols, vals


class _NS:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def sharded_maxcut_ops(n_global, deg, seed, rank, world, dev, group=None):
    """Row block `rank` of the MaxCut operators of a seeded random graph on n_global
    vertices: the local C rows (remapped, with their halo plan), the diagonal
    constraints of the owned rows, b = 1. The object carries what
    ``alm.AlmCore`` reads (problem.m, cop.con, c_mat.cpat, b, diag_aval)."""
    from .linops import ConstraintCSR, DevicePattern, padded

    b = block_bounds(n_global, world)
    lo, hi = b[rank], b[rank + 1]
    nown = hi - lo
    eu, ev = random_graph_edges(n_global, deg, seed, dev.dev)
    indptr, cols, vals = maxcut_rows(n_global, eu, ev, lo, hi)
    n_edges = int(eu.numel())
    del eu, ev
    plan = HaloPlan(lo, hi, indptr, cols, b, rank, world, group)
    pad_ptr = torch.zeros(nown + 1 + 16, dtype=I64, device=dev.dev)
    pad_ptr[:nown + 1] = indptr
    cpat = DevicePattern(nown, pad_ptr[:nown + 1], padded(plan.local_indices), padded(vals),
                         None, None, None)
    cpat.halo = plan if world > 1 else None
    ones = torch.ones(nown, dtype=torch.float64, device=dev.dev)
    empty_i = torch.zeros(0, dtype=I32, device=dev.dev)
    con = ConstraintCSR(m=nown, indptr=torch.arange(nown + 1, dtype=I64, device=dev.dev),
                        colidx=empty_i, pi=empty_i, pj=empty_i, val=ones, diag_aval=ones)
    problem = _NS(n=nown, m=nown, n_global=n_global, nnz_a_full=lambda: n_global)
    return _NS(problem=problem, cop=_NS(con=con), c_mat=_NS(cpat=cpat), b=ones.clone(),
               diag_aval=ones, is_diag=True, dev=dev, plan=plan, lo=lo, hi=hi, n_edges=n_edges)


# ---------------------------------------------------------------------------
# row-sharded solve of a diagonal-constraint problem (MaxCut family)
# ---------------------------------------------------------------------------

class ShardProblem:
    """Local view of a global SdpProblem on one rank: local sizes, global norms.

    ``n``/``m`` are the owned rows / constraints (buffer sizes of the solver
    stages); every normalisation (b norms, ||vec C||_1, nnz(A)) stays global,
    as do ``n_global``/``m_global`` for the rank rules (driver.py:130-135)."""

    def __init__(self, p, lo, hi):
        self.n = self.m = hi - lo
        self.n_global, self.m_global = p.n, p.m
        self.lo, self.hi = lo, hi
        self.b_norm1, self.b_norminf, self.c_vec_norm1 = p.b_norm1, p.b_norminf, p.c_vec_norm1
        self._nnz_a_full = p.nnz_a_full()
        self.maximize = p.maximize

    def nnz_a_full(self):
        return self._nnz_a_full


def slice_pattern(pat, lo, hi, bounds, rank, world, group, con_lo=None, halo=True):
    """Rows [lo, hi) of a DevicePattern, columns remapped through a HaloPlan.

    Adjoint rows keep their constraint coefficients; constraint ids are
    shifted by ``con_lo`` (they must belong to this rank's constraints)."""
    from .linops import DevicePattern, padded

    ptr = pat.indptr
    s0, s1 = int(ptr[lo]), int(ptr[hi])
    indptr = ptr[lo:hi + 1] - s0
    cols = pat.indices[s0:s1].to(I64)
    plan = HaloPlan(lo, hi, indptr, cols, bounds, rank, world, group)
    pad_ptr = torch.zeros(hi - lo + 1 + 16, dtype=I64, device=ptr.device)
    pad_ptr[:hi - lo + 1] = indptr
    cv = padded(pat.cv[s0:s1]) if pat.cv is not None else None
    at_ptr = at_con = at_val = None
    if pat.at_ptr is not None:
        a0, a1 = int(pat.at_ptr[s0]), int(pat.at_ptr[s1])
        ap = torch.zeros(s1 - s0 + 1 + 16, dtype=I64, device=ptr.device)
        ap[:s1 - s0 + 1] = pat.at_ptr[s0:s1 + 1] - a0
        at_ptr = ap[:s1 - s0 + 1]
        con = pat.at_con[a0:a1].to(I64) - (con_lo if con_lo is not None else 0)
        if con.numel() and (int(con.min()) < 0 or int(con.max()) >= hi - lo):
            raise NotImplementedError("row-sharded solve needs each constraint owned by the rank "
                                      "that owns its rows (diagonal constraints)")
        at_con = padded(con.to(I32))
        at_val = padded(pat.at_val[a0:a1])
    out = DevicePattern(hi - lo, pad_ptr[:hi - lo + 1], padded(plan.local_indices), cv, at_ptr, at_con, at_val)
    out.halo = plan if (halo and world > 1 and sum(plan.counts) > 0) else None
    return out


def build_sharded_operators(p, rank, world, dev, group=None):
    """Rank-local OperatorBundle of a diagonal-constraint problem (constraint c is
    a_c e_c e_c^T, e.g. MaxCut): factor rows, C/Omega/Omega_A pattern rows and
    constraints [lo, hi), remote columns through halo plans. Built from the
    single-device operators (linops.build_operators), then sliced."""
    from .linops import (AdjointOperator, CompressedOperator, ConstraintCSR, ObjectiveMatrix,
                         OperatorBundle, build_operators)

    full = build_operators(p, dev=dev)
    if not full.is_diag:
        raise NotImplementedError("row-sharded solve supports diagonal constraints (MaxCut family)")
    b = block_bounds(p.n, world)
    lo, hi = b[rank], b[rank + 1]
    cpat = slice_pattern(full.c_mat.cpat, lo, hi, b, rank, world, group)
    omega = slice_pattern(full.adj.omega, lo, hi, b, rank, world, group, con_lo=lo)
    apat = slice_pattern(full.adj.apat, lo, hi, b, rank, world, group, con_lo=lo)
    aval = full.diag_aval[lo:hi].clone()      # clone: slices of m-vectors must start 16-byte aligned
    fc = full.cop.con
    con = ConstraintCSR(m=hi - lo, indptr=(fc.indptr[lo:hi + 1] - fc.indptr[lo]).contiguous(),
                        colidx=fc.colidx[lo:hi], pi=fc.pi[lo:hi] - lo, pj=fc.pj[lo:hi] - lo,
                        val=fc.val[lo:hi].clone(), diag_aval=aval)
    sp = ShardProblem(p, lo, hi)
    cop = CompressedOperator(hi - lo, hi - lo, full.cop.ncols, full.cop.imap, full.cop.jmap,
                             full.cop.col_slot, con, dev)
    adj = AdjointOperator(hi - lo, hi - lo, full.adj.sup_i_host, full.adj.sup_j_host, omega, apat,
                          omega.cv, dev)
    ops = OperatorBundle(problem=sp, cop=cop, adj=adj, c_mat=ObjectiveMatrix(adj, cpat), dev=dev,
                         b=full.b[lo:hi].clone(), diag_aval=aval, omega_size_ref=full.omega_size_ref)
    ops.row_range = (lo, hi)
    del full
    return ops


def solve_sharded(p, cfg=None, *, group=None, dev=None):
    """driver.solve on this rank's row block; every rank returns the same report."""
    from . import driver
    from .device import default_device

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = dev or default_device()
    dev.world, dev.group = world, group
    ops = build_sharded_operators(p, rank, world, dev, group)
    return driver.solve(p, cfg, ops=ops)

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

import ctypes
import os

import numpy as np
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
    """In-place SUM over ranks, bit-identical on every rank and independent of the
    collective algorithm: the per-rank partials are all-gathered and added in rank
    order. (A backend's all-reduce may associate the sum differently on different
    ranks for three or more ranks; the solver branches on these scalars, so every
    rank must see the same bits.)"""
    world = dist.get_world_size(group)
    if world == 1:
        return t
    flat = t.reshape(-1)
    parts = _all_gather_1d(flat, world, group)                 # (world, count)
    acc = parts[0].clone()
    for r in range(1, world):
        acc += parts[r]
    flat.copy_(acc)
    return t


class HaloPlan:
    """Publish/receive plan of one contiguously partitioned index space (factor rows,
    or renumbered constraints) of a row-sharded solve.

    Built from a symmetric pattern's local CSR rows (``indptr``, global
    ``indices``): a row is published when it has a remote column. Or, with
    ``publish`` given, from an explicit list of local indices to publish.
    After construction ``local_indices`` holds the remapped int32 indices the
    kernels use, and ``remap`` maps any other global ids the same way:
    [0, nown) for owned ids, ``nown + r*maxb + t`` for the t-th published id
    of rank r -- the position that id lands at in the halo buffer.
    """

    def __init__(self, lo, hi, indptr, indices, bounds, rank, world, group=None, publish=None):
        self.lo, self.hi, self.rank, self.world, self.group = lo, hi, rank, world, group
        self.nown = nown = hi - lo
        self.bounds = bounds
        dev = indices.device
        indices = indices.to(I64)
        own = (indices >= lo) & (indices < hi)
        if publish is None:
            counts_row = (indptr[1:] - indptr[:-1]).to(I64)      # symmetric-pattern rule
            rows = torch.repeat_interleave(torch.arange(nown, device=dev, dtype=I64), counts_row)
            publish = torch.unique(rows[~own])                  # sorted local row ids
        else:
            publish = torch.unique(publish.to(device=dev, dtype=I64))
        nb = torch.tensor([publish.numel()], dtype=I64, device=dev)
        counts = _all_gather_1d(nb, world, group).view(-1)
        self.counts = counts.cpu().tolist()
        self.maxb = maxb = max(1, max(self.counts))
        padded = torch.full((maxb,), -1, dtype=I64, device=dev)
        padded[:publish.numel()] = publish + lo
        self.lists = _all_gather_1d(padded, world, group)        # (world, maxb) global ids, -1 padded
        self.publish = publish.to(I32).contiguous()             # local indices this rank sends
        if nown + world * maxb >= 2 ** 31:
            raise ValueError("owned block plus halo exceeds int32 indices")
        self.local_indices = self.remap(indices).to(I32).contiguous()
        self.halo_rows = world * maxb
        self._bufs = {}

    def remap(self, ids):
        """Global ids -> local/halo indices (int64); raises if a remote id is not published."""
        ids = ids.to(I64)
        lo, hi, maxb = self.lo, self.hi, self.maxb
        own = (ids >= lo) & (ids < hi)
        out = ids - lo
        remote = ids[~own]
        if remote.numel():
            bt = torch.tensor(self.bounds, dtype=I64, device=ids.device)
            owner = torch.searchsorted(bt, remote, right=True) - 1
            lists = self.lists.to(ids.device)
            keyed = torch.where(lists >= 0, lists, torch.full_like(lists, torch.iinfo(I64).max))
            pos = torch.empty_like(remote)
            for r in range(self.world):
                sel = owner == r
                if bool(sel.any()):
                    pos[sel] = torch.searchsorted(keyed[r].contiguous(), remote[sel])
            found = lists[owner, pos.clamp(max=maxb - 1)]
            if not bool((found == remote).all()):
                raise ValueError("a referenced remote index is missing from its owner's publish list "
                                 "(pattern not symmetric across the blocks)")
            out[~own] = self.nown + owner * maxb + pos
        return out

    def buffers(self, ld, like, slot=0):
        key = (ld, like.device, slot)
        b = self._bufs.get(key)
        if b is None:
            # a new leading dimension (rank escalation): the old rank's buffers are dead
            for k in [k for k in self._bufs if k[0] != ld]:
                del self._bufs[k]
            send = torch.zeros((self.maxb, ld), dtype=like.dtype, device=like.device)
            recv = torch.zeros((self.world * self.maxb, ld), dtype=like.dtype, device=like.device)
            b = self._bufs[key] = (send, recv)
        return b

    def exchange(self, X, ld, pack, slot=0):
        """Pack this rank's published rows of X and all-gather them; returns the halo buffer
        (one buffer per ``slot``, so several operands can be in flight at once)."""
        send, recv = self.buffers(ld, X, slot)
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


def _all_to_all_v(out, inp, out_splits, in_splits, group=None):
    """all_to_all_single with split sizes; CUDA tensors on gloo are staged through the host."""
    if inp.is_cuda and not _nccl(group):
        h_out = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(h_out, inp.cpu(), out_splits, in_splits, group=group)
        out.copy_(h_out)
        return out
    dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)
    return out


class PeerHaloPlan:
    """Point-to-point halo of one contiguously partitioned row space: rank r receives from
    each rank s exactly the rows of s that r's pattern rows reference (one all-to-all with
    split sizes), instead of every rank's whole publish list (HaloPlan's all-gather).

    On a uniformly random graph a rank's rows reference about half of any other block,
    while every row of it is referenced by some rank, so the all-gather moves (N-1)/N of
    the factor to every rank and this plan about half of that: half the NVLink bytes and
    half the receive buffer. Same interface as HaloPlan: ``local_indices`` (owned columns
    in [0, nown), remote column j at nown + its rank among this rank's needed ids -- the
    receive layout is ordered by owner, and the blocks are contiguous, so that is the sorted
    order), ``remap``, ``exchange``, ``halo_bytes``, ``halo_rows`` (receive rows), ``maxb``
    (send rows), ``counts`` (every rank's receive rows), ``publish`` (rows sent)."""

    def __init__(self, lo, hi, indptr, indices, bounds, rank, world, group=None):
        self.lo, self.hi, self.rank, self.world, self.group = lo, hi, rank, world, group
        self.nown = hi - lo
        self.bounds = bounds
        dev = indices.device
        indices = indices.to(I64)
        own = (indices >= lo) & (indices < hi)
        self.need = torch.unique(indices[~own])                       # sorted global ids
        bt = torch.tensor(bounds, dtype=I64, device=dev)
        owner = torch.searchsorted(bt, self.need, right=True) - 1
        recv = torch.bincount(owner, minlength=world).to(I64)
        send = torch.empty_like(recv)
        _all_to_all_v(send, recv, [1] * world, [1] * world, group)
        self.recv_counts = recv.cpu().tolist()
        self.send_counts = send.cpu().tolist()
        ids = torch.empty(sum(self.send_counts), dtype=I64, device=dev)
        _all_to_all_v(ids, self.need, self.send_counts, self.recv_counts, group)
        if ids.numel() and not bool(((ids >= lo) & (ids < hi)).all()):
            raise ValueError("peer halo: a rank requested rows outside this block")
        self.publish = (ids - lo).to(I32).contiguous()                # rows sent, destination-major
        self.halo_rows = int(sum(self.recv_counts))
        self.maxb = max(1, int(sum(self.send_counts)))
        tot = torch.tensor([self.halo_rows], dtype=I64, device=dev)
        self.counts = _all_gather_1d(tot, world, group).view(-1).cpu().tolist()
        if self.nown + self.halo_rows >= 2 ** 31:
            raise ValueError("owned block plus halo exceeds int32 indices")
        self.local_indices = self.remap(indices).to(I32).contiguous()
        self._bufs = {}

    def remap(self, ids):
        ids = ids.to(I64)
        own = (ids >= self.lo) & (ids < self.hi)
        out = ids - self.lo
        remote = ids[~own]
        if remote.numel():
            need = self.need.to(ids.device)
            pos = torch.searchsorted(need, remote).clamp(max=max(need.numel() - 1, 0))
            if need.numel() == 0 or not bool((need[pos] == remote).all()):
                raise ValueError("a referenced remote index is missing from this rank's peer halo")
            out[~own] = self.nown + pos
        return out

    def buffers(self, ld, like, slot=0):
        key = (ld, like.device, slot)
        b = self._bufs.get(key)
        if b is None:
            for k in [k for k in self._bufs if k[0] != ld]:
                del self._bufs[k]
            send = torch.zeros((max(1, self.publish.numel()), ld), dtype=like.dtype, device=like.device)
            recv = torch.zeros((max(1, self.halo_rows), ld), dtype=like.dtype, device=like.device)
            b = self._bufs[key] = (send, recv)
        return b

    def exchange(self, X, ld, pack, slot=0):
        """Pack the rows each peer needs (destination-major) and exchange them all-to-all."""
        send, recv = self.buffers(ld, X, slot)
        if self.publish.numel():
            pack(self.publish, X.reshape(-1, ld), send)
        _all_to_all_v(recv.view(-1)[:self.halo_rows * ld], send.view(-1)[:self.publish.numel() * ld],
                      [c * ld for c in self.recv_counts], [c * ld for c in self.send_counts], self.group)
        return recv

    def halo_bytes(self, ld):
        return self.halo_rows * ld * 8


# CL_MAX_PEERS / CL_PEER_ROW_BITS / CL_GHOST_PEERS of include/culorads.h
MAX_PEERS = 8
PEER_ROW_BITS = 28
GHOST_PEERS = -2

# halo mode of the diagonal-constraint (MaxCut-family) builders: "auto", "nvlink",
# "p2p" or "allgather" (make_halo_plan)
HALO_MODE = os.environ.get("CULORADS_HALO", "auto")


def peer_cols(owner, row):
    """CL_PEER_COL(owner, row) as int64 values of the int32 encoding (negative)."""
    return ((owner.to(I64) << PEER_ROW_BITS) | row.to(I64)) - (1 << 31)


def encode_peer_columns(ids, lo, hi, bounds):
    """Global column ids of rows [lo, hi) -> the peer-memory encoding: owned ids become
    local rows, remote ids CL_PEER_COL(owner, offset in the owner's block)."""
    ids = ids.to(I64)
    own = (ids >= lo) & (ids < hi)
    out = ids - lo
    remote = ids[~own]
    if remote.numel():
        bt = torch.tensor(bounds, dtype=I64, device=ids.device)
        owner = torch.searchsorted(bt, remote, right=True) - 1
        out[~own] = peer_cols(owner, remote - bt[owner])
    return out


def decode_peer_columns(enc, lo, bounds):
    """Inverse of encode_peer_columns (tests): encoded local indices -> global ids."""
    enc = enc.to(I64)
    out = enc + lo
    rem = enc < 0
    if bool(rem.any()):
        u = enc[rem] + (1 << 31)
        owner = (u >> PEER_ROW_BITS) & (MAX_PEERS - 1)
        row = u & ((1 << PEER_ROW_BITS) - 1)
        bt = torch.tensor(bounds, dtype=I64, device=enc.device)
        out[rem] = bt[owner] + row
    return out


class NvlinkHaloPlan:
    """Peer-memory ghost rows: no halo buffer and no collective moving factor rows.

    A remote column of this rank's pattern rows is encoded in its int32 index as
    ``CL_PEER_COL(owner, row)`` (row = the id's offset in the owner's block), and the SpMM
    loads that factor row in place from the owner GPU's memory (NVLink loads, issued by the
    same warps and in the same slot order as the local gathers, so remote and local traffic
    overlap tile by tile and the product is bit-identical to the halo paths). Each rank maps
    the peers' device allocations once (CUDA IPC, ``cl_ipc_export``/``cl_ipc_import``); per
    product only the (handle, offset) of every rank's operand is exchanged on the host (a
    gloo side group, no device sync), between two stream-ordered fences: ``exchange`` waits
    until every rank's operand is complete, ``release`` until every rank's product has
    read it (an 8-byte NCCL all-reduce on the compute stream; a host barrier on gloo).

    Replaces the all-gather / all-to-all of HaloPlan / PeerHaloPlan for the factor rows of C,
    Omega and Omega_A of diagonal-constraint (MaxCut) and single-entry (matrix completion)
    problems: the SpMM and the constraint kernel decode the same encoding. ``ghost_nown`` (= CL_GHOST_PEERS)
    is what goes into cl_pattern.nown; ``exchange`` returns the host table of peer addresses
    (cl_pattern.ghost)."""

    ghost_nown = GHOST_PEERS

    def __init__(self, lo, hi, indptr, indices, bounds, rank, world, group=None):
        if world > MAX_PEERS:
            raise ValueError(f"peer-memory halo supports at most {MAX_PEERS} ranks")
        if max(bounds[k + 1] - bounds[k] for k in range(world)) >= 2 ** PEER_ROW_BITS:
            raise ValueError("a row block exceeds the peer column encoding (2^28 rows)")
        self.lo, self.hi, self.rank, self.world, self.group = lo, hi, rank, world, group
        self.nown = hi - lo
        self.bounds = bounds
        indices = indices.to(I64)
        self.local_indices = self.remap(indices).to(I32).contiguous()
        nrem = torch.tensor([int(((indices < lo) | (indices >= hi)).sum())], dtype=I64, device=indices.device)
        self.counts = _all_gather_1d(nrem, world, group).view(-1).cpu().tolist()   # remote slots per rank
        self.remote_slots = self.counts[rank]
        self.halo_rows = 0
        self.maxb = 0
        self.publish = torch.zeros(0, dtype=I32, device=indices.device)
        self._obj_group = None
        self._fence_t = None
        self.stream = None           # the compute stream the products run on (Device.stream)
        self._imported = {}          # handle bytes -> mapped base address of a peer allocation
        self._tables = [(ctypes.c_uint64 * MAX_PEERS)() for _ in range(8)]   # >= 6 operands per launch
        self._tslot = 0

    def remap(self, ids):
        """Global ids -> local indices (int64 values of the int32 encoding)."""
        return encode_peer_columns(ids, self.lo, self.hi, self.bounds)

    # -- per product ---------------------------------------------------------
    def _objects(self):
        if self._obj_group is None:
            self._obj_group = (dist.new_group(list(range(self.world)), backend="gloo")
                               if _nccl(self.group) else self.group)
        return self._obj_group

    def fence(self, like):
        """Stream-ordered barrier over the ranks: work queued before it on every rank's
        compute stream is complete when work queued after it starts."""
        if self.world == 1:
            return
        st = self.stream if self.stream is not None else torch.cuda.current_stream(like.device)
        if like.is_cuda and _nccl(self.group):
            if self._fence_t is None:
                self._fence_t = torch.zeros(1, dtype=torch.float64, device=like.device)
            with torch.cuda.stream(st):
                dist.all_reduce(self._fence_t, group=self.group)
        else:
            st.synchronize()
            dist.barrier(group=self.group)

    def exchange(self, X, ld, pack=None, slot=0):
        """Fence, then the host table of every rank's row block of X as mapped here."""
        from . import _lib
        lib = _lib.load(require_device=True)
        self.fence(X)
        h = (ctypes.c_uint8 * _lib.CL_IPC_HANDLE_BYTES)()
        off = ctypes.c_int64(0)
        _lib.check(lib.cl_ipc_export(ctypes.c_void_p(X.data_ptr()), h, ctypes.byref(off)), "cl_ipc_export")
        allinfo = [None] * self.world
        dist.all_gather_object(allinfo, (bytes(h), int(off.value)), group=self._objects())
        tab = self._tables[self._tslot]
        self._tslot = (self._tslot + 1) % len(self._tables)
        for k in range(MAX_PEERS):
            tab[k] = 0
        for k, (hb, o) in enumerate(allinfo):
            if k == self.rank:
                tab[k] = X.data_ptr()
                continue
            base = self._imported.get(hb)
            if base is None:
                bp = ctypes.c_void_p()
                buf = (ctypes.c_uint8 * len(hb)).from_buffer_copy(hb)
                _lib.check(lib.cl_ipc_import(buf, ctypes.byref(bp)), "cl_ipc_import")
                base = self._imported[hb] = int(bp.value)
            tab[k] = base + o
        return _HostTable(tab)

    def release(self, X):
        """Fence after a product that read the peers' rows (no rank may overwrite its rows
        while another rank's product can still read them)."""
        self.fence(X)

    def close(self):
        from . import _lib
        lib = _lib.load(require_device=True)
        for base in self._imported.values():
            lib.cl_ipc_close(ctypes.c_void_p(base))
        self._imported.clear()

    def halo_bytes(self, ld):
        """Bytes this rank reads from peers per product (remote slots x one row each)."""
        return self.remote_slots * ld * 8


class _HostTable:
    """cl_pattern.ghost of the peer-memory mode: a host array of CL_MAX_PEERS addresses."""

    def __init__(self, tab):
        self.tab = tab

    def data_ptr(self):
        return ctypes.addressof(self.tab)


def nvlink_available(rank, world, group=None, device=None):
    """Every rank on its own CUDA device with peer access to every other (NCCL group):
    the peer-memory halo can be used. The same answer on every rank."""
    if world == 1 or world > MAX_PEERS or not _nccl(group):
        return False
    if "expandable_segments:true" in os.environ.get("PYTORCH_CUDA_ALLOC_CONF", "").replace(" ", "").lower():
        return False       # cuMemMap-backed segments have no legacy CUDA IPC handle
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    idx = torch.tensor([dev.index], dtype=I64, device=dev)
    devs = _all_gather_1d(idx, world, group).view(-1).cpu().tolist()
    ok = len(set(devs)) == world and all(
        torch.cuda.can_device_access_peer(dev.index, d) for d in devs if d != dev.index)
    flag = torch.tensor([1 if ok else 0], dtype=I64, device=dev)
    return min(_all_gather_1d(flag, world, group).view(-1).cpu().tolist()) == 1


def make_halo_plan(lo, hi, indptr, indices, bounds, rank, world, group=None, mode="auto", peer_ok=False):
    """The halo plan of a symmetric pattern's row block: the all-gather plan (HaloPlan) or the
    point-to-point one (PeerHaloPlan), whichever receives fewer rows on the worst rank
    ("auto"; every rank takes the same decision). With ``peer_ok`` (a pattern only the SpMM
    reads), "nvlink" -- and "auto" when every rank has its own peer-accessible GPU -- gives
    the peer-memory plan (NvlinkHaloPlan) instead."""
    if mode is None:
        mode = HALO_MODE
    if world > 1 and peer_ok and (mode == "nvlink" or (
            mode == "auto" and indices.is_cuda and nvlink_available(rank, world, group, indices.device))):
        return NvlinkHaloPlan(lo, hi, indptr, indices, bounds, rank, world, group)
    if mode == "nvlink":
        mode = "auto"
    if mode == "allgather" or world == 1:
        return HaloPlan(lo, hi, indptr, indices, bounds, rank, world, group)
    peer = PeerHaloPlan(lo, hi, indptr, indices, bounds, rank, world, group)
    if mode == "p2p":
        return peer
    ag = HaloPlan(lo, hi, indptr, indices, bounds, rank, world, group)
    return peer if max(peer.counts) < world * ag.maxb else ag


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
    plan = make_halo_plan(lo, hi, indptr, cols, b, rank, world, group, mode=None, peer_ok=True)
    plan.stream = getattr(dev, "stream", None)
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


def slice_pattern(pat, lo, hi, bounds, rank, world, group, con_map=None, halo=True):
    """Rows [lo, hi) of a DevicePattern, columns remapped through a HaloPlan.

    Adjoint rows keep their coefficients; constraint ids go through
    ``con_map`` (global id -> local/halo multiplier index)."""
    from .linops import DevicePattern, padded

    ptr = pat.indptr
    s0, s1 = int(ptr[lo]), int(ptr[hi])
    indptr = ptr[lo:hi + 1] - s0
    cols = pat.indices[s0:s1].to(I64)
    plan = make_halo_plan(lo, hi, indptr, cols, bounds, rank, world, group)
    pad_ptr = torch.zeros(hi - lo + 1 + 16, dtype=I64, device=ptr.device)
    pad_ptr[:hi - lo + 1] = indptr
    cv = padded(pat.cv[s0:s1]) if pat.cv is not None else None
    at_ptr = at_con = at_val = None
    if pat.at_ptr is not None:
        a0, a1 = int(pat.at_ptr[s0]), int(pat.at_ptr[s1])
        ap = torch.zeros(s1 - s0 + 1 + 16, dtype=I64, device=ptr.device)
        ap[:s1 - s0 + 1] = pat.at_ptr[s0:s1 + 1] - a0
        at_ptr = ap[:s1 - s0 + 1]
        at_con = padded(con_map(pat.at_con[a0:a1].to(I64)).to(I32))
        at_val = padded(pat.at_val[a0:a1])
    out = DevicePattern(hi - lo, pad_ptr[:hi - lo + 1], padded(plan.local_indices), cv, at_ptr, at_con, at_val)
    out.halo = plan if (halo and world > 1 and sum(plan.counts) > 0) else None
    return out, plan


def is_diag_problem(p):
    """Constraint c is a_c e_c e_c^T for every c (MaxCut family): the check of
    linops.build_operators' diagonal fast path."""
    m = p.m
    return (m == p.n and p.a_val.size == m and np.array_equal(p.a_con, np.arange(m))
            and np.array_equal(p.a_row, p.a_con) and np.array_equal(p.a_col, p.a_con))


def build_sharded_diag_operators(p, rank, world, dev, group=None):
    """Rank-local operators of a diagonal-constraint problem (MaxCut family), built from
    this rank's own rows only: no global operator build, so per-rank device memory and
    setup time scale with the rank's share of C (BASELINE configs[4], n = 1.7e8 over 8).

    Produces the same patterns, halo plan and constraint rows as slicing the single-device
    operators (``build_sharded_operators``'s general path; tests/test_shard.py checks
    equality): Omega's rows [lo, hi) are C's mirrored entries of those rows plus the
    diagonal positions (the constraints), each diagonal slot carrying one adjoint entry
    (local constraint i, a_c); Omega_A is the diagonal alone; constraint c is owned by the
    rank of row c, so the owned constraints are the block's rows and no multiplier halo
    is needed."""
    from .linops import (AdjointOperator, CompressedOperator, ConstraintCSR, DevicePattern, ObjectiveMatrix,
                         OperatorBundle, _csr_ptr, padded)

    n = p.n
    b = block_bounds(n, world)
    lo, hi = b[rank], b[rank + 1]
    nown = hi - lo
    tdev = dev.dev
    F64 = torch.float64
    r, c, v = np.asarray(p.C.rows), np.asarray(p.C.cols), np.asarray(p.C.vals)
    sel1 = (r >= lo) & (r < hi)
    sel2 = (r != c) & (c >= lo) & (c < hi)                   # mirrored (c, r) of stored (r, c)
    rows = torch.as_tensor(np.concatenate([r[sel1], c[sel2]]).astype(np.int64)).to(tdev)
    cols = torch.as_tensor(np.concatenate([c[sel1], r[sel2]]).astype(np.int64)).to(tdev)
    vals = torch.as_tensor(np.concatenate([v[sel1], v[sel2]]).astype(np.float64)).to(tdev)
    ccodes = (rows - lo) * n + cols
    o = torch.argsort(ccodes)
    ccodes, vals = ccodes[o], vals[o]
    ar = torch.arange(nown, dtype=I64, device=tdev)
    dcodes = ar * n + (ar + lo)
    sup = torch.unique(torch.cat([ccodes, dcodes]), sorted=True)
    S = int(sup.numel())
    slot_c = torch.searchsorted(sup, ccodes)
    slot_d = torch.searchsorted(sup, dcodes)
    cv = padded(torch.zeros(S, dtype=F64, device=tdev))
    cv[slot_c] = vals
    sup_r, sup_c = sup // n, sup % n
    o_ptr = _csr_ptr(sup_r, nown)
    plan = make_halo_plan(lo, hi, o_ptr, sup_c, b, rank, world, group, mode=None, peer_ok=True)
    plan.stream = getattr(dev, "stream", None)
    aval = torch.as_tensor(np.ascontiguousarray(p.a_val[lo:hi], dtype=np.float64)).to(tdev)
    omega = DevicePattern(nown, o_ptr, padded(plan.local_indices), cv, _csr_ptr(slot_d, S),
                          padded(ar.to(I32)), padded(aval.clone()))
    cpat = DevicePattern(nown, _csr_ptr(ccodes // n, nown), padded(plan.remap(ccodes % n).to(I32)),
                         padded(vals), None, None, None)
    apat = DevicePattern(nown, _csr_ptr(ar, nown), padded(ar.to(I32)), None, _csr_ptr(ar, nown),
                         padded(ar.to(I32)), padded(aval.clone()))
    halo = plan if (world > 1 and sum(plan.counts) > 0) else None
    omega.halo = cpat.halo = halo
    apat.halo = None                                      # diagonal positions: row-local
    con = ConstraintCSR(m=nown, indptr=_csr_ptr(ar, nown), colidx=padded((ar + lo).to(I32)),
                        pi=ar.to(I32).contiguous(), pj=ar.to(I32).contiguous(), val=padded(aval.clone()),
                        diag_aval=aval)
    sp_ = ShardProblem(p, lo, hi)
    ids = (ar + lo).to(I32)
    cop = CompressedOperator(nown, nown, n, ids, ids, None, con, dev)
    adj = AdjointOperator(nown, nown, None, None, omega, apat, omega.cv, dev)
    n_diag_stored = int(np.count_nonzero(r == c))
    omega_ref = n if p.dense_c else p.C.nnz_full + (n - n_diag_stored)
    ops = OperatorBundle(problem=sp_, cop=cop, adj=adj, c_mat=ObjectiveMatrix(adj, cpat), dev=dev,
                         b=torch.as_tensor(np.ascontiguousarray(p.b[lo:hi], dtype=np.float64)).to(tdev),
                         diag_aval=aval, omega_size_ref=omega_ref)
    ops.row_range = (lo, hi)
    ops.con_range = (lo, hi)
    return ops


def is_single_entry_problem(p):
    """Every constraint is one stored entry a_c at its own position (a_c (e_r e_k^T + e_k e_r^T),
    or a_c e_r e_r^T): matrix completion's family (problem.py:410)."""
    m = p.m
    if not (p.a_con.size == m and np.array_equal(p.a_con, np.arange(m))):
        return False
    if m and not np.all(np.asarray(p.a_val) != 0.0):
        return False
    from .problem import n_unique
    return n_unique(np.asarray(p.a_row) * p.n + np.asarray(p.a_col)) == m


def build_sharded_single_entry_operators(p, rank, world, dev, group=None):
    """Rank-local operators of a single-entry-constraint problem (matrix completion), built
    from the rank's own rows and the constraints that touch them: no global operator build.

    The same patterns, plans, multiplier halo, renumbering and constraint rows as slicing
    the single-device operators (``build_sharded_operators(local=False)``; tested equal):
    constraint c at (r, k) has the positions (r, k) and (k, r) (one if r = k), ordered by
    code; it is owned by the rank of row r when c is even, of row k when odd (the general
    path's alternation over a constraint's positions); constraints are renumbered
    owner-major. The compressed-column ids of the constraint rows (``colidx``, used only
    by the host-API ``cop.apply``) are left local, and ``cop`` carries no global maps."""
    from .linops import (AdjointOperator, CompressedOperator, ConstraintCSR, DevicePattern, ObjectiveMatrix,
                         OperatorBundle, _csr_ptr, padded)

    n, m = p.n, p.m
    tdev = dev.dev
    F64 = torch.float64
    b = block_bounds(n, world)
    lo, hi = b[rank], b[rank + 1]
    nown = hi - lo
    bt = torch.tensor(b, dtype=I64, device=tdev)
    T = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to(device=tdev, dtype=dt)  # noqa: E731
    r, k, v = T(p.a_row, I64), T(p.a_col, I64), T(p.a_val, F64)
    c = torch.arange(m, device=tdev, dtype=I64)
    two = r != k
    # ownership and owner-major renumbering (build_sharded_operators' general rule)
    prow = torch.where(two & (c % 2 == 1), k, r)
    owner = torch.searchsorted(bt, prow, right=True) - 1
    counts = torch.bincount(owner, minlength=world)
    bm = [0] + torch.cumsum(counts, 0).cpu().tolist()
    order = torch.argsort(owner * m + c)
    new_id = torch.empty(m, dtype=I64, device=tdev)
    new_id[order] = c
    lo_m, hi_m = bm[rank], bm[rank + 1]
    owned = order[lo_m:hi_m]
    inb = lambda x: (x >= lo) & (x < hi)  # noqa: E731
    ro, ko = r[owned], k[owned]
    if not bool((inb(ro) | inb(ko)).all()):       # cannot happen: the owner holds one of the rows
        raise AssertionError("single-entry ownership")
    pub = torch.unique(new_id[owned[~(inb(ro) & inb(ko))]] - lo_m)
    # constraint positions in this rank's rows: (r, k) for r in block, (k, r) for k in block
    s1 = inb(r)
    s2 = two & inb(k)
    a_rows = torch.cat([r[s1], k[s2]])
    a_cols = torch.cat([k[s1], r[s2]])
    a_con = torch.cat([c[s1], c[s2]])
    a_val = torch.cat([v[s1], v[s2]])
    acode = (a_rows - lo) * n + a_cols
    oa = torch.argsort(acode)
    acode, a_con, a_val = acode[oa], a_con[oa], a_val[oa]
    # the objective's mirrored entries in this rank's rows
    cr, cc, cvv = np.asarray(p.C.rows), np.asarray(p.C.cols), np.asarray(p.C.vals)
    t1 = (cr >= lo) & (cr < hi)
    t2 = (cr != cc) & (cc >= lo) & (cc < hi)
    c_rows = T(np.concatenate([cr[t1], cc[t2]]), I64)
    c_cols = T(np.concatenate([cc[t1], cr[t2]]), I64)
    c_vals = T(np.concatenate([cvv[t1], cvv[t2]]), F64)
    ccode = (c_rows - lo) * n + c_cols
    oc = torch.argsort(ccode)
    ccode, c_vals = ccode[oc], c_vals[oc]
    # Omega rows: union of both supports; one adjoint entry per constraint position
    sup = torch.unique(torch.cat([acode, ccode]), sorted=True)
    S = int(sup.numel())
    cv = padded(torch.zeros(S, dtype=F64, device=tdev))
    cv[torch.searchsorted(sup, ccode)] = c_vals
    slot_a = torch.searchsorted(sup, acode)
    o_ptr = _csr_ptr(sup // n, nown)
    ref = new_id[a_con]
    mplan = HaloPlan(lo_m, hi_m, None, ref, bm, rank, world, group, publish=pub)
    oplan = make_halo_plan(lo, hi, o_ptr, sup % n, b, rank, world, group, mode=None, peer_ok=True)
    at_con = padded(mplan.remap(ref).to(I32))
    omega = DevicePattern(nown, o_ptr, padded(oplan.local_indices), cv, _csr_ptr(slot_a, S), at_con,
                          padded(a_val.clone()))
    a_ptr = _csr_ptr(acode // n, nown)
    aplan = make_halo_plan(lo, hi, a_ptr, acode % n, b, rank, world, group, mode=None, peer_ok=True)
    apat = DevicePattern(nown, a_ptr, padded(aplan.local_indices), None,
                         _csr_ptr(torch.arange(acode.numel(), device=tdev, dtype=I64), acode.numel()),
                         padded(mplan.remap(ref).to(I32)), padded(a_val.clone()))
    c_ptr = _csr_ptr(ccode // n, nown)
    cplan = make_halo_plan(lo, hi, c_ptr, ccode % n, b, rank, world, group, mode=None, peer_ok=True)
    cpat = DevicePattern(nown, c_ptr, padded(cplan.local_indices), padded(c_vals.clone()), None, None, None)
    for pat, plan in ((omega, oplan), (apat, aplan), (cpat, cplan)):
        plan.stream = getattr(dev, "stream", None)
        pat.halo = plan if (world > 1 and sum(plan.counts) > 0) else None
    for pat in (omega, apat):
        pat.mhalo = mplan if (world > 1 and sum(mplan.counts) > 0) else None
    # owned constraint rows: positions in code order, remapped through the Omega halo
    two_o = two[owned]
    lens = torch.where(two_o, 2, 1).to(I64)
    ptr = torch.zeros(hi_m - lo_m + 1, dtype=I64, device=tdev)
    ptr[1:] = torch.cumsum(lens, 0)
    first_r = torch.minimum(ro, ko)            # code order: the smaller row first
    first_c = torch.maximum(ro, ko)
    pi = torch.stack([first_r, first_c], 1)
    pj = torch.stack([first_c, first_r], 1)
    keep = torch.stack([torch.ones_like(two_o), two_o], 1).reshape(-1)
    pi, pj = pi.reshape(-1)[keep], pj.reshape(-1)[keep]
    vv = torch.stack([v[owned], v[owned]], 1).reshape(-1)[keep]
    con = ConstraintCSR(m=hi_m - lo_m, indptr=ptr, colidx=padded(torch.zeros(pi.numel(), dtype=I32, device=tdev)),
                        pi=oplan.remap(pi).to(I32).contiguous(), pj=oplan.remap(pj).to(I32).contiguous(),
                        val=padded(vv), diag_aval=None)
    con.halo = oplan if world > 1 else None
    sp_ = ShardProblem(p, lo, hi)
    sp_.m = hi_m - lo_m
    K = int(m + int(two.sum()))
    cop = CompressedOperator(hi_m - lo_m, nown, K, None, None, None, con, dev)
    adj = AdjointOperator(hi_m - lo_m, nown, None, None, omega, apat, omega.cv, dev)
    omega_total = int(_all_gather_1d(torch.tensor([S], dtype=I64, device=tdev), world, group).sum())
    ops = OperatorBundle(problem=sp_, cop=cop, adj=adj, c_mat=ObjectiveMatrix(adj, cpat), dev=dev,
                         b=T(np.asarray(p.b), F64)[owned].clone(), diag_aval=None,
                         omega_size_ref=K if p.dense_c else omega_total)
    ops.row_range = (lo, hi)
    ops.con_range = (lo_m, hi_m)
    return ops


def build_sharded_operators(p, rank, world, dev, group=None, local=True):
    """Rank-local OperatorBundle of a row-sharded solve.

    Diagonal-constraint problems (MaxCut family) are built from the rank's own rows
    (``build_sharded_diag_operators``) unless ``local`` is False; other constraint
    families go through the general path below.

    Rows [lo, hi) of the factors and of the C/Omega/Omega_A patterns live on
    this rank. A constraint is owned by the rank of the smallest row among its
    positions, and every position must touch an owned row (diagonal
    constraints, matrix completion's symmetric pairs). Constraints are
    renumbered so that each rank's owned constraints form a contiguous block.
    Remote factor rows come through the Omega halo (constraint evaluation,
    SpMM), and the multipliers of constraints owned elsewhere come through a
    multiplier halo before each coefficient assembly. Built from the
    single-device operators (linops.build_operators), then sliced."""
    from .linops import (AdjointOperator, CompressedOperator, ConstraintCSR, ObjectiveMatrix,
                         OperatorBundle, build_operators, padded)

    if local and is_diag_problem(p):
        return build_sharded_diag_operators(p, rank, world, dev, group)
    if local and is_single_entry_problem(p):
        return build_sharded_single_entry_operators(p, rank, world, dev, group)
    full = build_operators(p, dev=dev)
    tdev = full.b.device
    b = block_bounds(p.n, world)
    lo, hi = b[rank], b[rank + 1]
    fc = full.cop.con
    m = p.m
    bt = torch.tensor(b, dtype=I64, device=tdev)

    # constraint ownership: the rank of one of its rows, alternating over the constraint's
    # positions (c mod nnz) so that e.g. completion's (j, n1+i) pairs spread over both blocks
    nnz_c = (fc.indptr[1:] - fc.indptr[:-1]).to(I64)
    cid = torch.repeat_interleave(torch.arange(m, device=tdev, dtype=I64), nnz_c)
    ar = torch.arange(m, device=tdev, dtype=I64)
    pick = fc.indptr[:-1].to(I64) + torch.remainder(ar, nnz_c.clamp(min=1))
    prow = fc.pi.to(I64)[pick.clamp(max=max(int(fc.pi.numel()) - 1, 0))] if fc.pi.numel() else ar
    owner = torch.where(nnz_c > 0, torch.searchsorted(bt, prow, right=True) - 1, ar * world // max(m, 1))
    counts = torch.bincount(owner, minlength=world)
    bm = [0] + torch.cumsum(counts, 0).cpu().tolist()
    # renumbering: owner-major, original order within an owner
    order = torch.argsort(owner * m + torch.arange(m, device=tdev, dtype=I64))
    new_id = torch.empty(m, dtype=I64, device=tdev)
    new_id[order] = torch.arange(m, device=tdev, dtype=I64)
    lo_m, hi_m = bm[rank], bm[rank + 1]
    owned = order[lo_m:hi_m]                                   # global ids, increasing

    # positions of owned constraints must touch an owned row
    sel = owner[cid] == rank
    pi_o, pj_o = fc.pi[sel].to(I64), fc.pj[sel].to(I64)
    touch = ((pi_o >= lo) & (pi_o < hi)) | ((pj_o >= lo) & (pj_o < hi))
    bad = torch.tensor([0 if bool(touch.all()) else 1], dtype=I64, device=tdev)
    if int(_all_gather_1d(bad, world, group).sum()) > 0:        # every rank raises together (no hang)
        raise NotImplementedError("row-sharded solve needs every position of a constraint to touch a row "
                                  "of the owning rank")
    # multiplier halo: owned constraints referenced from rows of other ranks
    outside = ~(((pi_o >= lo) & (pi_o < hi)) & ((pj_o >= lo) & (pj_o < hi)))
    pub = torch.unique(new_id[cid[sel][outside]] - lo_m)
    om = full.adj.omega
    s0, s1 = int(om.indptr[lo]), int(om.indptr[hi])
    a0, a1 = int(om.at_ptr[s0]), int(om.at_ptr[s1])
    ref = new_id[om.at_con[a0:a1].to(I64)]
    mplan = HaloPlan(lo_m, hi_m, None, ref, bm, rank, world, group, publish=pub)

    def con_map(c):
        return mplan.remap(new_id[c])

    cpat, _ = slice_pattern(full.c_mat.cpat, lo, hi, b, rank, world, group)
    omega, oplan = slice_pattern(om, lo, hi, b, rank, world, group, con_map=con_map)
    apat, _ = slice_pattern(full.adj.apat, lo, hi, b, rank, world, group, con_map=con_map)
    for pat in (omega, apat):
        pat.mhalo = mplan if (world > 1 and sum(mplan.counts) > 0) else None

    if full.is_diag:
        aval = full.diag_aval[owned].clone()       # clone: m-vector slices must start 16-byte aligned
    else:
        aval = None
    # owned constraint rows, positions remapped through the Omega row halo
    starts = fc.indptr[owned]
    lens = nnz_c[owned]
    ptr = torch.zeros(hi_m - lo_m + 1, dtype=I64, device=tdev)
    ptr[1:] = torch.cumsum(lens, 0)
    gather = torch.repeat_interleave(starts - ptr[:-1], lens) + torch.arange(int(ptr[-1]), device=tdev,
                                                                            dtype=I64)
    con = ConstraintCSR(m=hi_m - lo_m, indptr=ptr, colidx=padded(fc.colidx[gather]),
                        pi=oplan.remap(fc.pi[gather]).to(I32).contiguous(),
                        pj=oplan.remap(fc.pj[gather]).to(I32).contiguous(),
                        val=padded(fc.val[gather]), diag_aval=aval)
    con.halo = oplan if world > 1 and not full.is_diag else None
    sp = ShardProblem(p, lo, hi)
    sp.m = hi_m - lo_m
    cop = CompressedOperator(hi_m - lo_m, hi - lo, full.cop.ncols, full.cop.imap, full.cop.jmap,
                             full.cop.col_slot, con, dev)
    adj = AdjointOperator(hi_m - lo_m, hi - lo, None, None, omega, apat,
                          omega.cv, dev)
    ops = OperatorBundle(problem=sp, cop=cop, adj=adj, c_mat=ObjectiveMatrix(adj, cpat), dev=dev,
                         b=full.b[owned].clone(), diag_aval=aval, omega_size_ref=full.omega_size_ref)
    ops.row_range = (lo, hi)
    ops.con_range = (lo_m, hi_m)
    del full
    return ops


def solve_sharded(p, cfg=None, *, group=None, dev=None):
    """driver.solve on this rank's row block; every rank returns the same report.

    With ``cfg.reorder`` the rows are first relabelled in the locality order (as the
    1-GPU solve does); the report's U/V/lam are then this rank's block in that labelling
    and ``report.perm`` maps it back (row k is the caller's row perm[k])."""
    from . import driver
    from .device import Device

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    # a dedicated device context (never the process-wide default one): its scalar fetches
    # all-reduce over the group and its solve skips the 1-GPU-only native loops; a caller's
    # context gets its own world/group back on exit
    dev = dev or Device()
    saved = (dev.world, dev.group)
    dev.world, dev.group = world, group
    try:
        return _solve_sharded(p, cfg, group, dev, world, rank, driver)
    finally:
        dev.world, dev.group = saved


def _solve_sharded(p, cfg, group, dev, world, rank, driver):
    cfg = cfg or driver.SolverConfig()
    solve_p, perm = p, None
    if cfg.reorder:
        # the locality order (reorder.py) is computed identically on every rank; contiguous
        # row blocks of a mesh in this order touch only neighbouring blocks, so halos shrink
        # from most of the factor to the band at the block boundaries
        from . import reorder
        order = reorder.locality_order(p)
        if reorder.locality_gain(p, order) >= 2.0:
            solve_p, _ = reorder.permute(p, order)
            perm = order
    ops = build_sharded_operators(solve_p, rank, world, dev, group)
    if perm is not None:
        ops.perm = perm
    return driver.solve(p, cfg, ops=ops)


# ---------------------------------------------------------------------------
# per-rank device memory of a row-sharded solve
# ---------------------------------------------------------------------------

def halo_buffer_rows(ops):
    """Rows of halo receive/send buffers a rank's operators allocate per leading dimension:
    every distinct plan (C/Omega row halos: one buffer slot per SpMM operand in flight; the
    constraint halo of non-diagonal constraints: one slot per distinct operand of the line
    search, R and D)."""
    plans = {}
    for pat, slots in ((ops.c_mat.cpat, 1), (ops.adj.omega, 1), (ops.adj.apat, 1)):
        h = getattr(pat, "halo", None)
        if h is not None:
            plans[id(h)] = (h, max(slots, plans.get(id(h), (h, 0))[1]))
    h = getattr(ops.cop.con, "halo", None)
    if h is not None:
        plans[id(h)] = (h, max(2, plans.get(id(h), (h, 0))[1]))
    return sum(slots * (h.halo_rows + h.maxb) for h, slots in plans.values())


def _peer_rows(n_loc, world, deg):
    import math
    return int((world - 1) * n_loc * (1.0 - math.exp(-max(deg, 0.0) / world)))


def memory_model(n_global, world, r, nnz_c_per_row, m_global=None, nnz_a_per_con=1.0, halo_frac=1.0,
                 memory=8, halo_slots=1, pair=False, peer=False, nvlink=False):
    """Per-rank device bytes of a row-sharded solve at rank r.

    * stage buffers: driver.stage_factor_buffers(memory, pair) factors of n_loc x ld fp64
      (the ALM stage dominates: 2 memory + 8 = 24 at the default L-BFGS memory 8, + 2 for
      the pair buffer of single-entry constraints);
    * halo: ``halo_slots`` receive buffers of world * maxb rows plus the send buffer,
      maxb = halo_frac * n_loc published rows (random graphs: every row has a remote
      neighbour, halo_frac ~ 1; locality-ordered meshes: only the block-boundary band).
      ``peer``: the point-to-point plan (PeerHaloPlan) on a uniformly random pattern of
      nnz_c_per_row - 1 neighbours per row: each rank receives, and sends, the
      1 - exp(-deg/world) share of every other block that it references;
      ``nvlink``: the peer-memory plan (NvlinkHaloPlan) -- remote rows are read in place,
      no halo buffer;
    * operators: C rows (int32 index + fp64 value per nonzero, int64 row pointer), Omega
      (index, value, adjoint pointer per slot; constraint id + coefficient per adjoint
      entry), Omega_A and the constraint rows;
    * 16 m-vectors of the owned constraints.
    Returns a dict of byte counts and their total."""
    from .device import padded_ld
    from .driver import stage_factor_buffers
    m_global = n_global if m_global is None else m_global
    ld = padded_ld(r)
    n_loc = -(-n_global // world)
    m_loc = -(-m_global // world)
    nnz_c = n_loc * nnz_c_per_row
    nnz_a = m_loc * nnz_a_per_con
    factor = 8 * n_loc * ld
    maxb = int(halo_frac * n_loc)
    out = {
        "n_per_rank": n_loc, "ld": ld, "factor_bytes": factor,
        "stage_buffers": stage_factor_buffers(memory, pair) * factor,
        "halo": ((halo_slots + 1) * _peer_rows(n_loc, world, nnz_c_per_row - 1) if peer
                 else halo_slots * (world * maxb) + maxb) * ld * 8 if world > 1 and not nvlink else 0,
        "operators": (nnz_c * 12 + n_loc * 8) + (nnz_c + 2 * nnz_a) * 20 + nnz_a * 12 * 2 + nnz_a * 28
                     + m_loc * 8 + 2 * n_loc * 8,
        "m_vectors": 16 * 8 * m_loc,
    }
    out["total"] = sum(v for k, v in out.items() if k not in ("n_per_rank", "ld", "factor_bytes"))
    return out


# ---------------------------------------------------------------------------
# hooks of the native loops (cl_dist_hooks, include/culorads.h)
# ---------------------------------------------------------------------------

class _RawRows:
    """A device factor known only by its address (what HaloPlan.exchange needs of it)."""

    def __init__(self, addr, ld, like):
        self.addr, self.ld = addr, ld
        self.dtype, self.device, self.is_cuda = like.dtype, like.device, like.is_cuda

    def reshape(self, *shape):
        return self

    def data_ptr(self):
        return self.addr


def native_hooks(dev, ops):
    """cl_dist_hooks for cl_alm_inner_diag / cl_admm_step_diag on a row-sharded solve, or
    None on one GPU. ``exchange`` is C's halo exchange (the only pattern with remote
    columns in the diagonal-constraint loops); ``reduce`` is Device.fetch's rank-ordered
    all-reduce of a slab range into the pinned host mirror."""
    if dev.world == 1:
        return None
    import ctypes
    import sys
    import traceback

    from . import _lib
    plan = getattr(ops.c_mat.cpat, "halo", None)
    slab0, host0 = dev.slab.data_ptr(), dev.host.data_ptr()

    def exchange(ctx, xptr, ld):
        try:
            if plan is None:           # no remote column on any rank: the ghost block is never read
                return xptr
            return plan.exchange(_RawRows(xptr, ld, dev.slab), ld, dev.gather_rows).data_ptr()
        except Exception:             # noqa: BLE001 -- reported, then surfaced as CL_EARG by the loop
            traceback.print_exc(file=sys.stderr)
            return None

    def reduce(ctx, sptr, hptr, count, stream):
        try:
            so, ho = (sptr - slab0) // 8, (hptr - host0) // 8
            red = all_reduce_sum(dev.slab[so:so + count].clone(), dev.group)
            dev.host[ho:ho + count].copy_(red, non_blocking=True)
            dev.stream.synchronize()
            return 0
        except Exception:             # noqa: BLE001
            traceback.print_exc(file=sys.stderr)
            return 1

    def release(ctx, stream):
        try:
            plan.release(dev.slab)
            return 0
        except Exception:             # noqa: BLE001
            traceback.print_exc(file=sys.stderr)
            return 1

    h = _lib.DistHooks()
    h.ctx = None
    h.exchange = _lib.EXCHANGE_FN(exchange)
    h.reduce = _lib.REDUCE_FN(reduce)
    h.nown = getattr(plan, "ghost_nown", plan.nown) if plan is not None else int(ops.problem.n)
    peer = plan is not None and hasattr(plan, "release")
    h.release = _lib.RELEASE_FN(release) if peer else _lib.RELEASE_FN()
    h._keep = (h.exchange, h.reduce, h.release)   # the callbacks live as long as the struct
    return ctypes.pointer(h)

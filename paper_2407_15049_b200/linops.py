"""Fused, column-compressed constraint operators resident in HBM.

Device counterpart of the reference's lrsdp/linops.py. ``build_operators``
compresses the problem once (zero columns of the stacked operator removed,
Omega = union of constraint positions and the objective's support) and keeps
three CSR patterns over the n x n position grid on the device:

* ``omega``  -- the full support Omega: objective values cv[] plus, per slot,
  the adjoint row (constraint ids, coefficients). Every ``assemble(...)``
  of the reference (linops.py:177) is evaluated *inside* the SpMM kernel
  from these arrays -- the assembled matrix is never written to HBM.
* ``apat``   -- the constraint positions only (Omega_A): used when the
  objective does not participate (c_coeff = 0: the CG operator of
  admm.py:45 and the A*(w) R part of the gradient, alm.py:245).
* ``cpat``   -- the objective's own CSR (linops.py:274 symmetric_csr).

plus the constraint CSR (m rows, positions pre-resolved) for the fused
A(U V^T) kernel. Index arrays are int32, row pointers int64, values fp64.

The public classes (CompressedOperator, AdjointOperator, OperatorBundle,
spmm) accept numpy or torch operands and mirror the reference call surface.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import F64, I32, I64, default_device, padded_ld
from .exceptions import DimensionMismatchError
from .problem import SdpProblem


@dataclass
class DevicePattern:
    """CSR over positions with per-slot coefficient sources."""

    nrows: int
    indptr: torch.Tensor          # int64 [nrows+1]
    indices: torch.Tensor         # int32 [nnz]
    cv: torch.Tensor | None       # fp64  [nnz]   objective values
    at_ptr: torch.Tensor | None   # int64 [nnz+1] adjoint row per slot
    at_con: torch.Tensor | None   # int32
    at_val: torch.Tensor | None   # fp64

    scratch: torch.Tensor | None = None   # assembled slot coefficients (lazy)
    halo: object = None                   # shard.HaloPlan of a row-sharded pattern
    mhalo: object = None                  # shard.HaloPlan of the multipliers its adjoint rows read
    single_a: torch.Tensor | None = None  # Omega_A of single-entry constraints: a_c per slot

    @property
    def nnz(self):
        return int(self.indices.numel())

    def struct(self, c_coeff=None, w1=None, w2=None, use_cv=True, use_at=True):
        P = _lib.Pattern()
        P.nrows = self.nrows
        P.nnz = self.nnz
        P.indptr = self.indptr.data_ptr()
        P.indices = self.indices.data_ptr()
        if use_cv and self.cv is not None and c_coeff is not None:
            P.cv = self.cv.data_ptr()
            P.c_coeff = float(c_coeff)
        else:
            P.cv = None
            P.c_coeff = 0.0
        if use_at and self.at_ptr is not None and (w1 is not None or w2 is not None):
            P.at_ptr = self.at_ptr.data_ptr()
            P.at_con = self.at_con.data_ptr()
            P.at_val = self.at_val.data_ptr()
            P.w1 = w1.data_ptr() if w1 is not None else None
            P.w2 = w2.data_ptr() if w2 is not None else None
            if self.scratch is None:
                self.scratch = padded(torch.empty(self.nnz, dtype=F64, device=self.indices.device))
            P.scratch = self.scratch.data_ptr()
        else:
            P.at_ptr = P.at_con = P.at_val = P.w1 = P.w2 = None
            P.scratch = None
        return P

    def bytes(self):
        tot = 0
        for t in (self.indptr, self.indices, self.cv, self.at_ptr, self.at_con, self.at_val):
            if t is not None:
                tot += t.numel() * t.element_size()
        return tot


@dataclass
class ConstraintCSR:
    """Stacked constraint operator rows with resolved positions (pi, pj)."""

    m: int
    indptr: torch.Tensor   # int64 [m+1]
    colidx: torch.Tensor   # int32 compressed column k of each nonzero
    pi: torch.Tensor       # int32 row of the position
    pj: torch.Tensor       # int32 col of the position
    val: torch.Tensor      # fp64
    diag_aval: torch.Tensor | None = None   # set when constraint c is a_c e_c e_c^T (row-local)
    halo: object = None                      # shard.HaloPlan of the rows its positions reference


PAD = 16   # elements readable past the logical end (bulk copies read 16-byte supersets)


def padded(t):
    """Copy of ``t`` in an allocation PAD elements longer (zero tail); returns the logical view."""
    t = t.contiguous()
    buf = torch.zeros(t.numel() + PAD, dtype=t.dtype, device=t.device)
    buf[:t.numel()] = t
    return buf[:t.numel()]


# ---------------------------------------------------------------------------
# factor transfer helpers
# ---------------------------------------------------------------------------

def to_factor(W, dev=None, ld=None):
    """n x r operand (numpy or torch) -> padded contiguous device n x ld fp64."""
    dev = dev or default_device()
    if isinstance(W, torch.Tensor) and W.is_cuda and W.dtype == F64 and W.dim() == 2 and \
            W.is_contiguous() and (ld is None or W.shape[1] == ld) and W.shape[1] % 2 == 0:
        return W
    W = torch.as_tensor(np.asarray(W) if not isinstance(W, torch.Tensor) else W)
    if W.dim() != 2:
        raise DimensionMismatchError(f"factor must be 2-D, got shape {tuple(W.shape)}")
    n, r = W.shape
    ld = ld or padded_ld(r)
    out = torch.zeros((n, ld), dtype=F64, device=dev.dev)
    if r:
        out[:, :r] = W.to(device=dev.dev, dtype=F64)
    return out


def to_vec(x, dev=None):
    dev = dev or default_device()
    if isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == F64 and x.is_contiguous():
        return x
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(dev.dev)


def _host(t, like):
    """Return t as the caller's flavour: numpy for numpy inputs."""
    if isinstance(like, torch.Tensor):
        return t
    return t.detach().cpu().numpy()


# ---------------------------------------------------------------------------
# operators (reference call surface)
# ---------------------------------------------------------------------------

class CompressedOperator:
    """m x K stacked operator over retained positions (linops.py:115)."""

    def __init__(self, m, n, K, imap, jmap, col_slot, con, dev):
        self.m, self.n, self.ncols = m, n, K
        self.imap, self.jmap, self.col_slot = imap, jmap, col_slot
        self.con = con
        self.dev = dev
        # constraint rows as a pattern over compressed columns, for apply(x)
        self._rows = DevicePattern(m, con.indptr, con.colidx, con.val, None, None, None)

    def _check_pair(self, U, V):
        su = tuple(U.shape)
        sv = tuple(V.shape)
        if len(su) != 2 or len(sv) != 2 or su[0] != self.n or sv[0] != self.n or su[1] != sv[1]:
            raise DimensionMismatchError(f"factors must both be {self.n} x r, got {su} and {sv}")

    def outer_product(self, U, V):
        """x[k] = U[imap[k]] . V[jmap[k]] (linops.py:126), never forming U V^T."""
        self._check_pair(U, V)
        r = U.shape[1]
        ld = padded_ld(r)
        Ud, Vd = to_factor(U, self.dev, ld), to_factor(V, self.dev, ld)
        x = torch.empty(self.ncols, dtype=F64, device=self.dev.dev)
        self.dev.sddmm(self.imap, self.jmap, ld, Ud, Vd, x)
        return _host(x, U)

    def apply(self, xvals):
        """rows @ x (linops.py:139)."""
        if tuple(xvals.shape) != (self.ncols,):
            raise DimensionMismatchError(
                f"compressed vector has length {tuple(xvals.shape)}, operator has {self.ncols} columns")
        xd = to_vec(xvals, self.dev)
        out = torch.empty(self.m, dtype=F64, device=self.dev.dev)
        self.dev.spmm(self._rows, xd, 1, out=out, c_coeff=1.0)
        return _host(out, xvals)

    def apply_pair_dev(self, Ud, Vd, ld, out=None):
        if out is None:
            out = torch.empty(self.m, dtype=F64, device=self.dev.dev)
        self.dev.constraint_eval(self.con, ld, Ud, Vd, out)
        return out

    def apply_pair(self, U, V):
        """Fused A(U V^T) (linops.py:147)."""
        self._check_pair(U, V)
        ld = padded_ld(U.shape[1])
        out = self.apply_pair_dev(to_factor(U, self.dev, ld), to_factor(V, self.dev, ld), ld)
        return _host(out, U)


class AssembledMatrix:
    """c_coeff*C + A*(lam) + A*(extra) on Omega, evaluated lazily inside SpMM."""

    def __init__(self, adj, lam, extra, c_coeff):
        self.adj = adj
        self.lam = None if lam is None else to_vec(lam, adj.dev)
        self.extra = None if extra is None else to_vec(extra, adj.dev)
        self.c_coeff = float(c_coeff)
        self.shape = (adj.n, adj.n)

    def _pattern(self):
        # the objective-free form lives on Omega_A only (zeros elsewhere)
        if self.c_coeff == 0.0:
            return self.adj.apat, None
        return self.adj.omega, self.c_coeff

    def matmul_dev(self, Xd, ld, out=None, alpha=1.0, Y=(), ycoef=()):
        pat, cc = self._pattern()
        if out is None:
            out = torch.empty((self.adj.n, ld), dtype=F64, device=self.adj.dev.dev)
        self.adj.dev.spmm(pat, Xd, ld, alpha=alpha, out=out, Y=Y, ycoef=ycoef, c_coeff=cc,
                          w1=self.lam, w2=self.extra)
        return out

    def __matmul__(self, V):
        return spmm(self, V)

    def values(self):
        """Slot values (sup order), for inspection/tests."""
        data = torch.zeros(self.adj.size, dtype=F64, device=self.adj.dev.dev)
        if self.lam is not None:
            data += self.adj.apply_dev(self.lam)
        if self.extra is not None:
            data += self.adj.apply_dev(self.extra)
        if self.c_coeff != 0.0:
            data += self.c_coeff * self.adj.c_vals
        return data

    def toarray(self):
        S = np.zeros(self.shape)
        S[self.adj.sup_i_host, self.adj.sup_j_host] = self.values().cpu().numpy()
        return S


class AdjointOperator:
    """Support-aligned transpose rows plus objective values (linops.py:153)."""

    def __init__(self, m, n, sup_i, sup_j, omega, apat, c_vals, dev):
        """``sup_i``/``sup_j`` (host position arrays of Omega) may be None: they are then
        derived from the device CSR on first use (inspection/toarray only -- the solve
        never needs Omega's positions on the host)."""
        self.m, self.n = m, n
        self._sup = (sup_i, sup_j) if sup_i is not None else None
        self.omega, self.apat = omega, apat
        self.c_vals = c_vals
        self.dev = dev
        self._atrows = DevicePattern(omega.nnz, omega.at_ptr, omega.at_con, omega.at_val,
                                     None, None, None)

    def _support(self):
        if self._sup is None:
            om = self.omega
            counts = (om.indptr[1:] - om.indptr[:-1]).to(I64)
            rows = torch.repeat_interleave(torch.arange(om.nrows, device=counts.device, dtype=I64), counts)
            self._sup = (rows.cpu().numpy(), om.indices[:om.nnz].to(I64).cpu().numpy())
        return self._sup

    @property
    def sup_i_host(self):
        return self._support()[0]

    @property
    def sup_j_host(self):
        return self._support()[1]

    @property
    def sup_i(self):
        return self.sup_i_host

    @property
    def sup_j(self):
        return self.sup_j_host

    @property
    def size(self):
        return self.omega.nnz

    def apply_dev(self, yd):
        out = torch.empty(self.size, dtype=F64, device=self.dev.dev)
        self.dev.spmm(self._atrows, yd, 1, out=out, c_coeff=1.0)
        return out

    def apply(self, y):
        """At @ y on the support (linops.py:170)."""
        if tuple(y.shape) != (self.m,):
            raise DimensionMismatchError(f"multiplier has shape {tuple(y.shape)}, expected ({self.m},)")
        return _host(self.apply_dev(to_vec(y, self.dev)), y)

    def assemble(self, lam=None, extra=None, c_coeff=1.0):
        """Lazy c_coeff*C + A*(lam) + A*(extra) (linops.py:177)."""
        for v in (lam, extra):
            if v is not None and tuple(v.shape) != (self.m,):
                raise DimensionMismatchError(f"multiplier has shape {tuple(v.shape)}, expected ({self.m},)")
        return AssembledMatrix(self, lam, extra, c_coeff)


def spmm(S, V):
    """Assembled n x n matrix times n x r factor (linops.py:199)."""
    if S.shape[1] != V.shape[0]:
        raise DimensionMismatchError(f"cannot multiply {S.shape} by {tuple(V.shape)}")
    r = V.shape[1]
    ld = padded_ld(r)
    dev = S.adj.dev
    out = S.matmul_dev(to_factor(V, dev, ld), ld)
    res = out[:, :r]
    return res if isinstance(V, torch.Tensor) else res.cpu().numpy()


class ObjectiveMatrix(AssembledMatrix):
    """C alone, over its own CSR (linops.py:274 symmetric_csr)."""

    def __init__(self, adj, cpat):
        self.adj = adj
        self.lam = self.extra = None
        self.c_coeff = 1.0
        self.shape = (adj.n, adj.n)
        self.cpat = cpat

    def _pattern(self):
        return self.cpat, 1.0


@dataclass
class OperatorBundle:
    """Problem data plus the device operators (linops.py:283)."""

    problem: SdpProblem
    cop: CompressedOperator
    adj: AdjointOperator
    c_mat: ObjectiveMatrix
    dev: object
    b: torch.Tensor             # device b
    diag_aval: torch.Tensor | None   # set when constraint c is a_c e_c e_c^T (MaxCut)
    omega_size_ref: int              # |Omega| as the reference reports it

    @property
    def is_diag(self):
        return self.diag_aval is not None

    def objective_value(self, U, V):
        """<C, U V^T> as <C V, U> (linops.py:292)."""
        r = U.shape[1]
        ld = padded_ld(r)
        Ud, Vd = to_factor(U, self.dev, ld), to_factor(V, self.dev, ld)
        return objective_dev(self, Ud, Vd, ld)

    def device_bytes(self):
        tot = self.adj.omega.bytes() + self.adj.apat.bytes() + self.c_mat.cpat.bytes()
        con = self.cop.con
        tot += sum(t.numel() * t.element_size() for t in (con.indptr, con.colidx, con.pi, con.pj, con.val))
        return tot


def objective_dev(ops, Ud, Vd, ld, at=0, fetch=True):
    dev = ops.dev
    dev.spmm(ops.c_mat.cpat, Vd, ld, out=None, Z=[Ud], dots=[("out", ("z", 0))], at=at, c_coeff=1.0)
    if fetch:
        return float(dev.fetch(at + 1)[at])
    return None


def operator_stats(cop, adj):
    return {"K": cop.ncols, "omega_size": adj.size, "nnz_rows": int(cop.con.val.numel()),
            "dense_c": False}


# ---------------------------------------------------------------------------
# compression on the device
# ---------------------------------------------------------------------------

def _csr_ptr(rows, nrows):
    ptr = torch.zeros(nrows + 1 + PAD, dtype=I64, device=rows.device)
    if rows.numel():
        ptr[1:nrows + 1] = torch.cumsum(torch.bincount(rows, minlength=nrows), 0)
    return ptr[:nrows + 1]


def _mirror(n, tag, r, c, v):
    off = r != c
    return (torch.cat([r * n + c, c[off] * n + r[off]]), torch.cat([tag, tag[off]]),
            torch.cat([v, v[off]]))


def build_operators(p: SdpProblem, dense_c=None, dev=None) -> OperatorBundle:
    """Compress ``p`` into device-resident operators (linops.py:216 + :297)."""
    dev = dev or default_device()
    n, m = p.n, p.m
    if n >= 2 ** 31 - 1:
        raise ValueError("n must fit int32 indices")
    T = lambda a, dt: dev.put(np.asarray(a), dtype=dt)  # noqa: E731
    a_row, a_col, a_con, a_val = (T(p.a_row, I64), T(p.a_col, I64), T(p.a_con, I64),
                                  T(p.a_val, F64))
    codes, cons, vals = _mirror(n, a_con, a_row, a_col, a_val)
    uniq, colidx = torch.unique(codes, sorted=True, return_inverse=True)
    K = int(uniq.numel())
    imap, jmap = uniq // n, uniq % n

    # constraint CSR, rows sorted by compressed column (scipy canonical order)
    order = torch.argsort(cons * max(K, 1) + colidx)
    ccol = colidx[order]
    con = ConstraintCSR(m=m, indptr=_csr_ptr(cons, m), colidx=padded(ccol.to(I32)),
                        pi=imap[ccol].to(I32).contiguous(), pj=jmap[ccol].to(I32).contiguous(),
                        val=padded(vals[order]))

    c_r, c_c, c_v = T(p.C.rows, I64), T(p.C.cols, I64), T(p.C.vals, F64)
    ccodes, _, cvals = _mirror(n, torch.zeros_like(c_r), c_r, c_c, c_v)
    sup = torch.unique(torch.cat([uniq, ccodes]), sorted=True)
    S = int(sup.numel())
    slot_a = torch.searchsorted(sup, uniq)
    slot_c = torch.searchsorted(sup, ccodes)
    cv = padded(torch.zeros(S, dtype=F64, device=dev.dev))
    cv[slot_c] = cvals
    sup_i, sup_j = sup // n, sup % n

    # adjoint rows aligned to Omega: entries (slot of column, constraint) sorted
    s_of = slot_a[colidx]
    o2 = torch.argsort(s_of * max(m, 1) + cons)
    at_ptr = _csr_ptr(s_of, S)
    omega = DevicePattern(n, _csr_ptr(sup_i, n), padded(sup_j.to(I32)), cv, at_ptr,
                          padded(cons[o2].to(I32)), padded(vals[o2]))

    # Omega_A: the K constraint positions only (same entry order, by column)
    o3 = torch.argsort(colidx * max(m, 1) + cons)
    apat = DevicePattern(n, _csr_ptr(imap, n), padded(jmap.to(I32)), None, _csr_ptr(colidx, K),
                         padded(cons[o3].to(I32)), padded(vals[o3]))

    # objective's own CSR
    o4 = torch.argsort(ccodes)
    cs = ccodes[o4]
    cpat = DevicePattern(n, _csr_ptr(cs // n, n), padded((cs % n).to(I32)), padded(cvals[o4]),
                         None, None, None)

    # single-entry constraints (each A_c = a_c (e_i e_j^T + e_j e_i^T) or a_c e_i e_i^T, and no
    # two constraints share a position): the ADMM operator fuses into one pass over Omega_A
    # (cl_single_entry_apply). Matrix completion (problem.py:410) has this shape.
    single = None
    nnz_c = con.indptr[1:] - con.indptr[:-1]
    apc = apat.at_ptr[1:] - apat.at_ptr[:-1]
    if m and bool(((nnz_c == 1) | (nnz_c == 2)).all()) and bool((apc == 1).all()):
        st = con.indptr[:-1]
        pi0, pj0 = con.pi.to(I64)[st], con.pj.to(I64)[st]
        two = nnz_c == 2
        nxt = (st + 1).clamp(max=max(int(con.pi.numel()) - 1, 0))
        pi1, pj1 = con.pi.to(I64)[nxt], con.pj.to(I64)[nxt]
        ok1 = (~two) & (pi0 == pj0)
        ok2 = two & (pi0 == pj1) & (pj0 == pi1) & (pi0 != pj0) & (con.val[st] == con.val[nxt])
        if bool((ok1 | ok2).all()):
            single = padded(apat.at_val[apat.at_ptr[:-1]].contiguous())
    apat.single_a = single

    cop = CompressedOperator(m, n, K, imap.to(I32), jmap.to(I32), slot_a, con, dev)
    adj = AdjointOperator(m, n, None, None, omega, apat, cv, dev)      # Omega stays on the device

    diag = None
    if (m == n and p.a_val.size == m and np.array_equal(p.a_con, np.arange(m))
            and np.array_equal(p.a_row, p.a_con) and np.array_equal(p.a_col, p.a_con)):
        diag = a_val.contiguous()
        con.diag_aval = diag

    if dense_c is None:
        dense_c = p.dense_c
    omega_ref = K if dense_c else S
    return OperatorBundle(problem=p, cop=cop, adj=adj, c_mat=ObjectiveMatrix(adj, cpat), dev=dev,
                          b=T(p.b, F64), diag_aval=diag, omega_size_ref=omega_ref)


def symmetric_csr(M):
    """Host CSR of a SymmetricSparse (linops.py:274), for callers that want scipy."""
    import scipy.sparse as sp
    off = M.rows != M.cols
    r = np.concatenate([M.rows, M.cols[off]])
    c = np.concatenate([M.cols, M.rows[off]])
    v = np.concatenate([M.vals, M.vals[off]])
    return sp.csr_matrix((v, (r, c)), shape=(M.n, M.n))


def compress(p: SdpProblem, dense_c=None):
    """(CompressedOperator, AdjointOperator) pair (linops.py:216)."""
    ops = build_operators(p, dense_c=dense_c)
    return ops.cop, ops.adj

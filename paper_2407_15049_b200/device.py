"""Device runtime: stream, reduction workspace, scalar slab, kernel launchers.

torch supplies device memory and the stream (plumbing only); every compute
launch goes through libculorads (``_lib``). Reductions land in a device
"scalar slab"; the host reads a prefix of it with one pinned copy + stream
sync at each decision point of the algorithm (``fetch``).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import CL_MAXDOT, CL_MAXIN, CL_MAXY, CL_OUT, check

F64 = torch.float64
I32 = torch.int32
I64 = torch.int64

SLAB = 4096


def ptr(t):
    """Raw device address of a tensor (or None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def padded_ld(r):
    """Leading dimension of an n x r factor: r rounded up to even (16-byte rows)."""
    return max(2, r + (r & 1))


class Device:
    """Per-solve device context (one CUDA stream, one workspace)."""

    def __init__(self, device=None):
        self.lib = _lib.load(require_device=True)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.dev = torch.device(device)
        self.stream = torch.cuda.current_stream(self.dev)
        self.ws = torch.zeros(_lib.CL_WS_ALLOC, dtype=F64, device=self.dev)
        self.slab = torch.zeros(SLAB, dtype=F64, device=self.dev)
        self.host = torch.zeros(SLAB, dtype=F64, pin_memory=True)
        self.launches = 0
        self.group = None          # torch.distributed group of a row-sharded solve (shard.py)
        self.world = 1

    # -- plumbing ---------------------------------------------------------
    @property
    def sp(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    def slot(self, k, count=1):
        """Device pointer to slab[k:k+count]."""
        return ctypes.c_void_p(self.slab.data_ptr() + 8 * k)

    def fetch(self, count):
        """Copy slab[:count] to the host (pinned) and wait; returns numpy view.

        In a row-sharded solve every slab entry is a per-rank partial sum: the
        prefix is all-reduced (into a copy, the partials stay) first, so all
        ranks read identical scalars."""
        if self.world > 1:
            from .shard import all_reduce_sum
            red = all_reduce_sum(self.slab[:count].clone(), self.group)
            self.host[:count].copy_(red, non_blocking=True)
            self.stream.synchronize()
            return self.host[:count].numpy()
        self.host[:count].copy_(self.slab[:count], non_blocking=True)
        self.stream.synchronize()
        return self.host[:count].numpy()

    def zeros(self, *shape):
        return torch.zeros(*shape, dtype=F64, device=self.dev)

    def empty(self, *shape):
        return torch.empty(*shape, dtype=F64, device=self.dev)

    def put(self, a, dtype=F64):
        a = np.ascontiguousarray(a)
        return torch.as_tensor(a).to(device=self.dev, dtype=dtype, non_blocking=False)

    # -- launches ---------------------------------------------------------
    def lincomb(self, out, ins, coefs, dots=None, at=0, mode=_lib.CL_DOT_PAIRS, N=None):
        """out = sum coefs[j]*ins[j]; dots -> slab[at:].

        dots: list of (a, b) operand pairs (mode PAIRS; use 'out' or input index),
        or True for modes OUT_ALL / FIRST_TWO.
        """
        a = _lib.LincombArgs()
        a.nin = len(ins)
        a.mode = mode
        if len(ins) > CL_MAXIN:
            raise ValueError("too many operands")
        for j, (t, c) in enumerate(zip(ins, coefs)):
            a.inp[j] = t.data_ptr()
            a.coef[j] = float(c)
        a.out = out.data_ptr() if out is not None else None
        ndot = 0
        if mode == _lib.CL_DOT_PAIRS and dots:
            for d, (x, y) in enumerate(dots):
                a.da[d] = CL_OUT if x == "out" else x
                a.db[d] = CL_OUT if y == "out" else y
            ndot = len(dots)
        elif dots:
            ndot = 1
        a.ndot = ndot
        if N is None:
            N = (out if out is not None else ins[0]).numel()
        rc = self.lib.cl_lincomb(ctypes.byref(a), int(N), self.slot(at) if ndot else None,
                                 ptr(self.ws) if ndot else None, self.sp)
        self.launches += 1
        check(rc, "cl_lincomb")

    def spmm(self, pat, X, ld, alpha=1.0, out=None, Y=(), ycoef=(), Z=(), dots=None, at=0,
             c_coeff=None, w1=None, w2=None, use_cv=True, use_at=True, drow=None, dmul=None):
        """out = alpha * S X + sum ycoef*Y [+ diag(drow*dmul) Y[0]] over a device pattern
        (see linops.DevicePattern)."""
        P = pat.struct(c_coeff=c_coeff, w1=w1, w2=w2, use_cv=use_cv, use_at=use_at)
        e = _lib.Epilogue()
        e.drow = drow.data_ptr() if drow is not None else None
        e.dmul = dmul.data_ptr() if dmul is not None else None
        e.ny = len(Y)
        for j, (t, c) in enumerate(zip(Y, ycoef)):
            e.Y[j] = t.data_ptr()
            e.ycoef[j] = float(c)
        e.nz = len(Z)
        for j, t in enumerate(Z):
            e.Z[j] = t.data_ptr()
        nd = 0
        if dots:
            for d, (x, y) in enumerate(dots):
                e.da[d] = _op_code(x)
                e.db[d] = _op_code(y)
            nd = len(dots)
        e.ndot = nd
        halo = getattr(pat, "halo", None)
        if halo is not None:
            ghost = halo.exchange(X, ld, self.gather_rows)
            P.ghost = ghost.data_ptr()
            P.nown = getattr(halo, "ghost_nown", halo.nown)
        mhalo = getattr(pat, "mhalo", None)
        if mhalo is not None and (w1 is not None or w2 is not None) and P.at_ptr:
            # multipliers of constraints owned by other ranks (row-sharded solve)
            if w1 is not None:
                P.w1g = mhalo.exchange(w1, 1, self.gather_rows, slot=0).data_ptr()
            if w2 is not None:
                P.w2g = mhalo.exchange(w2, 1, self.gather_rows, slot=1).data_ptr()
            P.mown = mhalo.nown
        rc = self.lib.cl_pattern_spmm(ctypes.byref(P), ptr(X), int(ld), float(alpha), ctypes.byref(e),
                                      ptr(out), self.slot(at) if nd else None,
                                      ptr(self.ws) if nd else None, self.sp)
        self.launches += 1
        check(rc, "cl_pattern_spmm")
        self._release(halo, X)

    def constraint_eval(self, con, ld, X1, Y1, out1, X2=None, Y2=None, X3=None, Y3=None, out2=None):
        if con.diag_aval is not None:
            rc = self.lib.cl_diag_constraint_eval(int(con.m), ptr(con.diag_aval), int(ld), ptr(X1), ptr(Y1),
                                                  ptr(X2), ptr(Y2), ptr(out1), ptr(X3), ptr(Y3), ptr(out2),
                                                  self.sp)
            self.launches += 1
            check(rc, "cl_diag_constraint_eval")
            return
        halo = getattr(con, "halo", None)
        if halo is not None:
            # remote factor rows of the owned constraints' positions, one halo per distinct operand
            ops_ = [X1, Y1, X2, Y2, X3, Y3]
            seen, ghosts = {}, []
            for t in ops_:
                if t is None:
                    ghosts.append(None)
                    continue
                key = id(t)       # object identity: the same on every rank (data_ptr is 0 for empty tensors)
                if key not in seen:
                    seen[key] = halo.exchange(t, ld, self.gather_rows, slot=len(seen))
                ghosts.append(seen[key])
            garr = (ctypes.c_void_p * 6)(*[g.data_ptr() if g is not None else None for g in ghosts])
            rc = self.lib.cl_constraint_eval_halo(int(con.m), ptr(con.indptr), ptr(con.pi), ptr(con.pj),
                                                  ptr(con.val), int(ld), ptr(X1), ptr(Y1), ptr(X2), ptr(Y2),
                                                  ptr(out1), ptr(X3), ptr(Y3), ptr(out2), garr,
                                                  int(getattr(halo, "ghost_nown", halo.nown)), self.sp)
            self.launches += 1
            check(rc, "cl_constraint_eval_halo")
            self._release(halo, X1)
            return
        rc = self.lib.cl_constraint_eval(int(con.m), ptr(con.indptr), ptr(con.pi), ptr(con.pj),
                                         ptr(con.val), int(ld), ptr(X1), ptr(Y1), ptr(X2), ptr(Y2),
                                         ptr(out1), ptr(X3), ptr(Y3), ptr(out2), self.sp)
        self.launches += 1
        check(rc, "cl_constraint_eval")

    def diag_cg_apply(self, aval, ld, rho, p, Wf, Q, r=None, beta=0.0, at=0):
        """[p <- r + beta p]; Q = rho (A*(A(p Wf^T)) Wf + p) for diagonal A; <p, Q> -> slab[at]."""
        rc = self.lib.cl_diag_cg_apply(int(p.shape[0]), int(ld), ptr(aval), float(rho), float(beta), ptr(r),
                                       ptr(p), ptr(Wf), ptr(Q), self.slot(at), ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_diag_cg_apply")

    def diag_cg_apply_rows(self, aval, ld, rho, p, Wf, coef, r=None, beta=0.0, at=0):
        """diag_cg_apply writing the per-row coefficients rho a_c y_c to coef (n doubles) instead of Q."""
        rc = self.lib.cl_diag_cg_apply_rows(int(p.shape[0]), int(ld), ptr(aval), float(rho), float(beta), ptr(r),
                                            ptr(p), ptr(Wf), ptr(coef), self.slot(at), ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_diag_cg_apply_rows")

    def diag_cg_step(self, ld, rho, coef, Wf, x_in, x_out, p, r, alpha=0.0, qr=0.0, pq_at=None, at=0):
        """CG update with Q = coef Wf + rho p rebuilt per row; alpha = qr / slab[pq_at] on the
        device when pq_at is given; <r, r> -> slab[at]."""
        rc = self.lib.cl_diag_cg_step(int(p.shape[0]), int(ld), float(rho), ptr(coef), ptr(Wf), float(alpha),
                                      float(qr), None if pq_at is None else self.slot(pq_at), ptr(x_in), ptr(x_out),
                                      ptr(p), ptr(r), self.slot(at), ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_diag_cg_step")

    def _halo_struct(self, pat, X, ld):
        P = pat.struct(c_coeff=1.0)
        halo = getattr(pat, "halo", None)
        if halo is not None:
            P.ghost = halo.exchange(X, ld, self.gather_rows).data_ptr()
            P.nown = getattr(halo, "ghost_nown", halo.nown)
        return P

    @staticmethod
    def _release(halo, X):
        """Peer-memory ghosts (shard.NvlinkHaloPlan): fence after the product that read them."""
        if halo is not None and hasattr(halo, "release"):
            halo.release(X)

    def diag_admm_cg_init(self, cpat, Wf, x0, ld, scale, rho, nlam, aval, r, at, cw=None):
        """Fused rhs + initial CG residual (cl_diag_admm_cg_init); ||rhs||^2, ||r||^2 -> slab[at:at+2];
        C Wf itself -> cw when given."""
        P = self._halo_struct(cpat, Wf, ld)
        rc = self.lib.cl_diag_admm_cg_init(ctypes.byref(P), ptr(Wf), ptr(x0), int(ld), float(scale), float(rho),
                                           ptr(nlam), ptr(aval), ptr(r), ptr(cw), self.slot(at), ptr(self.ws),
                                           self.sp)
        self.launches += 1
        check(rc, "cl_diag_admm_cg_init")
        self._release(getattr(cpat, "halo", None), Wf)

    def diag_admm_step_end(self, cpat, U, V, ld, aval, b, lam, rho, ax, lam_new, at):
        """Fused objective / A(UV^T) / residual / dual ascent (cl_diag_admm_step_end) -> slab[at:at+3]."""
        P = self._halo_struct(cpat, V, ld)
        rc = self.lib.cl_diag_admm_step_end(ctypes.byref(P), ptr(U), ptr(V), int(ld), ptr(aval), ptr(b), ptr(lam),
                                            float(rho), ptr(ax), ptr(lam_new), self.slot(at), ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_diag_admm_step_end")
        self._release(getattr(cpat, "halo", None), V)

    def diag_admm_step_end_rows(self, CU, U, V, ld, aval, b, lam, rho, ax, lam_new, at):
        """Step end from a stored C U (cl_diag_admm_step_end_rows): <CU, V>, ||ax - b||^2,
        lam_new . b -> slab[at:at+3]."""
        rc = self.lib.cl_diag_admm_step_end_rows(int(U.shape[0]), int(ld), ptr(CU), ptr(U), ptr(V), ptr(aval), ptr(b),
                                                 ptr(lam), float(rho), ptr(ax), ptr(lam_new), self.slot(at),
                                                 ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_diag_admm_step_end_rows")

    def single_entry_apply(self, apat, ld, W, Wf, rho, out, at=0):
        """Fused half-step operator for single-entry constraints; <W, out> -> slab[at]."""
        rc = self.lib.cl_single_entry_apply(int(apat.nrows), ptr(apat.indptr), ptr(apat.indices), ptr(apat.single_a),
                                            int(ld), ptr(W), ptr(Wf), float(rho), ptr(out), self.slot(at),
                                            ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_single_entry_apply")

    def single_entry_apply_pair(self, apat, ld, P2, rho, out, at=0):
        """single_entry_apply with W and Wf interleaved in the pair buffer P2 (n x 2ld)."""
        rc = self.lib.cl_single_entry_apply_pair(int(apat.nrows), ptr(apat.indptr), ptr(apat.indices),
                                                 ptr(apat.single_a), int(ld), ptr(P2), float(rho), ptr(out),
                                                 self.slot(at), ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_single_entry_apply_pair")

    def constraint_eval_pair(self, con, ld, P2, out1, out2):
        """Line-search products from the pair buffer P2 = [R | D]: out1 = A(RD^T + DR^T), out2 = A(DD^T)."""
        rc = self.lib.cl_constraint_eval_pair(int(con.m), ptr(con.indptr), ptr(con.pi), ptr(con.pj), ptr(con.val),
                                              int(ld), ptr(P2), ptr(out1), ptr(out2), self.sp)
        self.launches += 1
        check(rc, "cl_constraint_eval_pair")

    def pair_pack(self, X, ld, P2, half):
        """P2[:, half*ld:(half+1)*ld] = X."""
        rc = self.lib.cl_pair_pack(int(X.shape[0]), int(ld), ptr(X), ptr(P2), int(half), self.sp)
        self.launches += 1
        check(rc, "cl_pair_pack")

    def cg_direction_pair(self, ld, beta, r, p, P2):
        """p = r + beta p, also into P2's first half."""
        rc = self.lib.cl_cg_direction_pair(int(p.shape[0]), int(ld), float(beta), ptr(r), ptr(p), ptr(P2), self.sp)
        self.launches += 1
        check(rc, "cl_cg_direction_pair")

    def cg_step_dev(self, qr, pq_at, x_in, x_out, p, r, Q, at=0):
        """x_out = x_in + alpha p; r -= alpha Q with alpha = qr / slab[pq_at] on the device;
        <r, r> -> slab[at] (update skipped for a non-finite or non-positive curvature)."""
        rc = self.lib.cl_cg_step_dev(int(r.numel()), float(qr), self.slot(pq_at), ptr(x_in), ptr(x_out), ptr(p),
                                     ptr(r), ptr(Q), self.slot(at), ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_cg_step_dev")

    def cg_step(self, alpha, x_in, x_out, p, r, Q, at=0):
        """x_out = x_in + alpha p; r -= alpha Q; <r, r> -> slab[at]."""
        rc = self.lib.cl_cg_step(int(r.numel()), float(alpha), ptr(x_in), ptr(x_out), ptr(p), ptr(r), ptr(Q),
                                 self.slot(at), ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_cg_step")

    def gather_rows(self, idx, X, out):
        """out[i] = X[idx[i]] (halo packing, shard.py)."""
        rc = self.lib.cl_gather_rows(ptr(idx), int(idx.numel()), int(out.shape[1]), ptr(X), ptr(out), self.sp)
        self.launches += 1
        check(rc, "cl_gather_rows")

    def sddmm(self, imap, jmap, ld, X, Y, out):
        rc = self.lib.cl_sddmm(int(imap.numel()), ptr(imap), ptr(jmap), int(ld), ptr(X), ptr(Y),
                               ptr(out), self.sp)
        self.launches += 1
        check(rc, "cl_sddmm")

    def diag_update(self, args, at=0):
        rc = self.lib.cl_diag_alm_update(ctypes.byref(args), self.slot(at), ptr(self.ws), self.sp)
        self.launches += 1
        check(rc, "cl_diag_alm_update")

    def basis_project(self, Q, kc, n, v, h):
        rc = self.lib.cl_basis_project(ptr(Q), int(Q.shape[1]), int(kc), int(n), ptr(v), ptr(h),
                                       ptr(self.ws), self.sp)
        self.launches += 2
        check(rc, "cl_basis_project")

    def basis_subtract(self, Q, kc, n, h, v):
        rc = self.lib.cl_basis_subtract(ptr(Q), int(Q.shape[1]), int(kc), int(n), ptr(h), ptr(v),
                                        self.sp)
        self.launches += 1
        check(rc, "cl_basis_subtract")


def _op_code(x):
    """Epilogue operand code: ('y', j) -> j, 'out' -> CL_OUT, ('z', j) -> 16 + j."""
    if x == "out":
        return CL_OUT
    kind, j = x
    if kind == "y":
        return j
    if kind == "z":
        return 16 + j
    raise ValueError(x)


_DEFAULT = {}


def default_device():
    """Process-wide Device for the current CUDA device (created lazily)."""
    key = torch.cuda.current_device()
    d = _DEFAULT.get(key)
    if d is None:
        d = Device()
        _DEFAULT[key] = d
    return d


assert CL_MAXDOT >= 48 and CL_MAXY == 4

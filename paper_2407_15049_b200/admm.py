"""Stage two: splitting ADMM on X = U V^T with matrix-free CG half-steps.

Device restatement of the reference's lrsdp/admm.py. Each half-step solves

    rho * A*(A(W Wf^T)) Wf + rho W = -scale*C Wf - A*(lam) Wf + rho A*(b) Wf + rho Wf

by CG (Algorithm 2). On the device the operator is one fused constraint
launch (A(W Wf^T) over the constraint nonzeros) plus one Omega_A pattern
product whose epilogue adds rho*W and reduces <p, Q>; the right-hand side
assembles -scale*C - A*(lam) + rho*A*(b) inside the SpMM coefficients.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from collections import deque
from dataclasses import dataclass

import torch

from .alm import DualVector
from .device import padded_ld
from .exceptions import DivergedError, SpdViolationError
from .linops import to_factor, to_vec


@dataclass
class CgWorkspace:
    """Tolerance and cap of one CG solve (admm.py:31)."""

    eps: float
    max_iter: int
    residual: object = None
    direction: object = None
    op_output: object = None

    def __post_init__(self):
        if not self.eps > 0:
            raise ValueError("CG tolerance must be positive")


class HalfStep:
    """Device buffers + the SPD operator of a half-step (admm.py:45)."""

    S_CG = 400       # slab offsets
    S_RHS = 410

    def __init__(self, ops, n, ld):
        self.ops, self.dev, self.n, self.ld = ops, ops.dev, n, ld
        m = ops.problem.m
        dev = self.dev
        self.y = dev.empty(m)
        self.r = dev.empty(n, ld)
        self.p = dev.empty(n, ld)
        self.Q = dev.empty(n, ld)
        self.coef = self.Q.view(-1)[:n]      # per-row CG coefficients (Q itself is not stored in the loop)
        self.cu = None
        self.nlam = dev.empty(m)
        self.rhob = dev.empty(m)

    def cu_buffer(self):
        """C U of the diagonal ADMM step (written by the V half-step's start, read by the step end)."""
        if self.cu is None:
            self.cu = self.dev.empty(self.n, self.ld)
        return self.cu

    def apply(self, W, Wf, rho, out, dot_with=None, at=None):
        """out = rho*(A*(A(W Wf^T)) Wf + W); optional <dot_with, out> -> slab[at]."""
        ops, dev = self.ops, self.dev
        if ops.is_diag and (dot_with is None or dot_with is W):
            # diagonal A: the whole operator is row-local, one streaming pass (cl_diag_cg_apply)
            dev.diag_cg_apply(ops.diag_aval, self.ld, rho, W, Wf, out, at=at if at is not None else 0)
            return out
        apat = ops.adj.apat
        if (apat.single_a is not None and apat.halo is None and self.ld <= 64
                and (dot_with is None or dot_with is W)):
            # single-entry constraints (matrix completion): A(W Wf^T) recomputed per slot, one pass
            dev.single_entry_apply(apat, self.ld, W, Wf, rho, out, at=at if at is not None else 0)
            return out
        dev.constraint_eval(ops.cop.con, self.ld, W, Wf, self.y)
        dots = [(("y", 0), "out")] if dot_with is not None else None
        dev.spmm(ops.adj.apat, Wf, self.ld, alpha=rho, out=out, Y=[W], ycoef=[rho], w1=self.y,
                 dots=dots, at=at if at is not None else 0)
        return out

    def rhs(self, Wf, lam, rho, scale, out, at):
        """out = S_b Wf + rho Wf with S_b = -scale C - A*(lam) + rho A*(b); ||out||^2 -> slab[at]."""
        ops, dev = self.ops, self.dev
        if ops.is_diag:
            # S_b = -scale C + diag(a (rho b - lam)): the C product plus a row-diagonal epilogue term
            dev.lincomb(self.nlam, [ops.b, lam], [rho, -1.0])
            dev.spmm(ops.c_mat.cpat, Wf, self.ld, alpha=-scale, out=out, Y=[Wf], ycoef=[rho], c_coeff=1.0,
                     drow=self.nlam, dmul=ops.diag_aval, dots=[("out", "out")], at=at)
            return out
        dev.lincomb(self.nlam, [lam], [-1.0])
        dev.lincomb(self.rhob, [ops.b], [rho])
        dev.spmm(ops.adj.omega, Wf, self.ld, alpha=1.0, out=out, Y=[Wf], ycoef=[rho],
                 c_coeff=-scale, w1=self.nlam, w2=self.rhob, dots=[("out", "out")], at=at)
        return out

    def cg(self, x, Wf, rho, rhs, eps, max_iter, x0=None):
        """admm.py:65 on device factors. Returns (iterations, residual).

        The iterate starts at ``x0`` (read only) when given and is written to
        ``x``; otherwise ``x`` is updated in place."""
        if self.ops.is_diag:
            return self._cg_diag(x, Wf, rho, rhs, eps, max_iter, x0)
        dev = self.dev
        if x0 is not None:
            dev.lincomb(x, [x0], [1.0])
        r, p, Q = self.r, self.p, self.Q
        A = self.S_CG
        self.apply(x, Wf, rho, Q)
        dev.lincomb(r, [rhs, Q], [1.0, -1.0], dots=[("out", "out")], at=A)
        qr = float(dev.fetch(A + 1)[A])
        rnorm = math.sqrt(qr)
        if rnorm <= eps:
            return 0, rnorm
        dev.lincomb(p, [r], [1.0])
        apat = self.ops.adj.apat
        # single-entry constraints: the CG direction and Wf share one pair buffer [p_i | Wf_i],
        # so each operator slot gathers one 2 ld run (bit-identical to the two-operand kernel)
        pair = (PAIR and apat.single_a is not None and apat.halo is None and self.ld <= 64)
        if pair:
            if getattr(self, "P2", None) is None:
                self.P2 = dev.empty(self.n, 2 * self.ld)
            dev.pair_pack(Wf, self.ld, self.P2, 1)
            dev.pair_pack(p, self.ld, self.P2, 0)
        its = 0
        for k in range(max_iter):
            if pair:
                dev.single_entry_apply_pair(apat, self.ld, self.P2, rho, Q, at=A + 1)
            else:
                self.apply(p, Wf, rho, Q, dot_with=p, at=A + 1)
            if dev.world == 1:
                # x += alpha p; r -= alpha Q; <r, r> with alpha = qr / <p, Q> taken on the device,
                # so <p, Q> and <r, r> come back in one read (a rejected curvature skips the update)
                dev.cg_step_dev(qr, A + 1, x, x, p, r, Q, at=A + 2)
                h = dev.fetch(A + 3)
                pq = float(h[A + 1])
            else:
                # row-sharded: <p, Q> is a per-rank partial until the slab is combined
                pq = float(dev.fetch(A + 2)[A + 1])
            if not math.isfinite(pq):
                raise DivergedError("CG produced non-finite curvature", last_iterate=x)
            if pq <= 0.0:
                raise SpdViolationError(f"non-positive curvature {pq:.3e} in CG (operator not SPD)")
            if dev.world > 1:
                dev.cg_step(qr / pq, x, x, p, r, Q, at=A + 2)
                h = dev.fetch(A + 3)
            qn = float(h[A + 2])
            rnorm = math.sqrt(qn)
            its = k + 1
            if rnorm <= eps:
                break
            if pair:
                dev.cg_direction_pair(self.ld, qn / qr, r, p, self.P2)
            else:
                dev.lincomb(p, [r, p], [1.0, qn / qr])
            qr = qn
        dev.lincomb(None, [x], [0.0], dots=[(0, 0)], at=A + 3)
        if not math.isfinite(float(dev.fetch(A + 4)[A + 3])):
            raise DivergedError("CG iterate diverged", last_iterate=x)
        return its, rnorm


    def _cg_diag(self, x, Wf, rho, rhs, eps, max_iter, x0):
        """Same iteration as ``cg`` for diagonal A with fused launches: the direction
        update p = r + beta p rides on the next operator application and the x/r
        updates share one pass (cl_diag_cg_apply, cl_cg_step)."""
        dev, ops = self.dev, self.ops
        r, p, Q = self.r, self.p, self.Q
        A = self.S_CG
        xs = x if x0 is None else x0
        dev.diag_cg_apply(ops.diag_aval, self.ld, rho, xs, Wf, Q, at=A)      # Q = apply(x0)
        dev.lincomb(r, [rhs, Q], [1.0, -1.0], dots=[("out", "out")], at=A)
        qr = float(dev.fetch(A + 1)[A])
        rnorm = math.sqrt(qr)
        if rnorm <= eps:
            if x0 is not None:
                dev.lincomb(x, [x0], [1.0])
            return 0, rnorm
        its = 0
        beta = 0.0
        for k in range(max_iter):
            dev.diag_cg_apply_rows(ops.diag_aval, self.ld, rho, p, Wf, self.coef, r=r, beta=beta, at=A + 1)
            pq = float(dev.fetch(A + 2)[A + 1])
            if not math.isfinite(pq):
                raise DivergedError("CG produced non-finite curvature", last_iterate=xs)
            if pq <= 0.0:
                raise SpdViolationError(f"non-positive curvature {pq:.3e} in CG (operator not SPD)")
            alpha = qr / pq
            dev.diag_cg_step(self.ld, rho, self.coef, Wf, xs, x, p, r, alpha=alpha, at=A + 2)
            xs = x
            qn = float(dev.fetch(A + 3)[A + 2])
            rnorm = math.sqrt(qn)
            its = k + 1
            if rnorm <= eps:
                break
            beta = qn / qr
            qr = qn
        if x0 is not None and its == 0:
            dev.lincomb(x, [x0], [1.0])
        dev.lincomb(None, [x], [0.0], dots=[(0, 0)], at=A + 3)
        if not math.isfinite(float(dev.fetch(A + 4)[A + 3])):
            raise DivergedError("CG iterate diverged", last_iterate=x)
        return its, rnorm


def subproblem_apply(W, W_fixed, rho, ops):
    """rho*(A*(A(W Wf^T)) Wf + W)  (admm.py:45)."""
    r = W.shape[1]
    ld = padded_ld(r)
    hs = HalfStep(ops, W.shape[0], ld)
    out = hs.apply(to_factor(W, ops.dev, ld), to_factor(W_fixed, ops.dev, ld), rho,
                   ops.dev.empty(W.shape[0], ld))
    out = out[:, :r]
    return out if isinstance(W, torch.Tensor) else out.cpu().numpy()


def subproblem_rhs(W_fixed, dual: DualVector, ops, scale=1.0, S_b=None):
    """Right-hand side of a half-step system (admm.py:52)."""
    r = W_fixed.shape[1]
    ld = padded_ld(r)
    hs = HalfStep(ops, W_fixed.shape[0], ld)
    out = ops.dev.empty(W_fixed.shape[0], ld)
    if S_b is not None:
        Wf = to_factor(W_fixed, ops.dev, ld)
        S_b.matmul_dev(Wf, ld, out=out, Y=[Wf], ycoef=[dual.rho])
    else:
        hs.rhs(to_factor(W_fixed, ops.dev, ld), to_vec(dual.lam, ops.dev), dual.rho, scale, out,
               at=HalfStep.S_RHS)
    out = out[:, :r]
    return out if isinstance(W_fixed, torch.Tensor) else out.cpu().numpy()


def cg_solve(x0, apply_op, rhs, ws: CgWorkspace):
    """CG with Frobenius products for an arbitrary operator callback (admm.py:65).

    Generic (host-orchestrated) form used by tests and callers with their own
    operator; the solver's hot path uses ``HalfStep.cg``. Operands may be
    numpy or device tensors; the vector algebra always runs on the device.
    """
    from .device import default_device
    dev = default_device()
    host = not isinstance(x0, torch.Tensor)
    shape = tuple(x0.shape)
    ld = padded_ld(shape[1]) if len(shape) == 2 else None

    def dv(a):
        if len(shape) == 2:
            return to_factor(a, dev, ld)
        return to_vec(a, dev).clone()

    def back(t):
        return t[:, :shape[1]] if len(shape) == 2 else t

    def op(t):
        res = apply_op(back(t) if not host else back(t).cpu().numpy())
        return dv(res)

    x = dv(x0).clone()
    b = dv(rhs)
    r = dev.empty(*x.shape)
    dev.lincomb(r, [b, op(x)], [1.0, -1.0], dots=[("out", "out")], at=420)
    qr = float(dev.fetch(421)[420])
    rnorm = math.sqrt(qr)
    if rnorm <= ws.eps:
        ws.residual = r
        return (back(x).cpu().numpy() if host else back(x)), 0, rnorm
    p = r.clone()
    its = 0
    for k in range(ws.max_iter):
        Q = op(p)
        dev.lincomb(None, [p, Q], [0.0, 0.0], dots=[(0, 1)], at=421)
        pq = float(dev.fetch(422)[421])
        if not math.isfinite(pq):
            raise DivergedError("CG produced non-finite curvature", last_iterate=x)
        if pq <= 0.0:
            raise SpdViolationError(f"non-positive curvature {pq:.3e} in CG (operator not SPD)")
        alpha = qr / pq
        dev.lincomb(x, [x, p], [1.0, alpha])
        dev.lincomb(r, [r, Q], [1.0, -alpha], dots=[("out", "out")], at=422)
        qn = float(dev.fetch(423)[422])
        rnorm = math.sqrt(qn)
        its = k + 1
        if rnorm <= ws.eps:
            break
        dev.lincomb(p, [r, p], [1.0, qn / qr])
        qr = qn
    if not bool(torch.isfinite(x).all()):
        raise DivergedError("CG iterate diverged", last_iterate=x)
    ws.residual, ws.direction = r, p
    return (back(x).cpu().numpy() if host else back(x)), its, rnorm


@dataclass
class AdmmState:
    """Factor halves (device n x ld), shared dual, cached A(U V^T) (admm.py:105)."""

    U: object
    V: object
    dual: DualVector
    ax: object = None
    r: int = 0

    def set_factors(self, U=None, V=None):
        if U is not None:
            self.U = U
        if V is not None:
            self.V = V
        self.ax = None

    def constraint_values(self, ops):
        if self.ax is None:
            ld = self.U.shape[1]
            self.ax = ops.cop.apply_pair_dev(self.U, self.V, ld)
        return self.ax


@dataclass
class StepStats:
    cg_iters_u: int
    cg_iters_v: int
    resid_u: float
    resid_v: float
    hit_cap: bool


def _resid(ops, ax, res, at):
    ops.dev.lincomb(res, [ax, ops.b], [1.0, -1.0], dots=[("out", "out")], at=at)


# single-entry constraints: CG operator on the pair buffer [p | Wf] (cl_single_entry_apply_pair)
PAIR = os.environ.get("CULORADS_PAIR", "1") != "0"
NATIVE = True     # diagonal constraints: run the step's control flow in C++ (row-sharded: with hooks)
NATIVE_GENERIC = True   # other constraint families on one GPU: cl_admm_step_generic
# Problems with at most this many row-lanes (n times the lanes that share a factor row,
# lanes_for(ld)) run each ADMM step as one cooperative launch (cl_admm_step_diag_fused):
# there, latency rather than HBM bounds the step (measured crossover).
FUSED = os.environ.get("CULORADS_FUSED", "1") != "0"
FUSED_MAX_LANES = int(os.environ.get("CULORADS_FUSED_MAX", 1 << 19))


def lanes_for(ld):
    """Lanes per factor row of the one-launch kernels (fused_rows.cuh lanes_for)."""
    h2 = max(ld // 2, 1)
    g = 1
    while g < h2 and g < 32:
        g *= 2
    return g


def _admm_step_native(state, ops, scale, cg_cap, cg_rel_floor, cg_primal_coeff, hs, pool):
    """admm_step through cl_admm_step_diag: the same launches as the Python branch below,
    with the scalar decisions taken in native code (bit-identical iterates)."""
    from . import _lib
    dev = ops.dev
    p = ops.problem
    n, ld = state.U.shape
    if getattr(hs, "r_v", None) is None:
        hs.r_v = dev.empty(n, ld)
    a = getattr(hs, "native_args", None)
    if a is None:
        # the fields that stay fixed over the steps of one HalfStep, set once (host time per
        # step matters at small n, where a step costs tens of microseconds)
        a = hs.native_args = _lib.AdmmDiagArgs()
        a.n, a.ld = n, ld
        a.aval, a.b = ops.diag_aval.data_ptr(), ops.b.data_ptr()
        a.r, a.r_v, a.p, a.Q = hs.r.data_ptr(), hs.r_v.data_ptr(), hs.p.data_ptr(), hs.Q.data_ptr()
        a.cu = hs.cu_buffer().data_ptr()
        a.nlam, a.res = hs.nlam.data_ptr(), hs.y.data_ptr()
        a.cpat = ops.c_mat.cpat.struct(c_coeff=1.0)
        a.binf = float(p.b_norminf)
        a.slab = dev.slot(470).value
        a.host = dev.host.data_ptr() + 8 * 470
        a.ws = dev.ws.data_ptr()
        a.stream = dev.stream.cuda_stream
    a.lam = state.dual.lam.data_ptr()
    lam_new = hs.lam_spare if getattr(hs, "lam_spare", None) is not None else dev.empty(p.m)
    a.lam_new = lam_new.data_ptr()
    if state.ax is None:
        ax = dev.empty(p.m)
        a.ax_valid = 0
    else:
        ax = state.ax
        a.ax_valid = 1
    known = getattr(state, "pnorm2_ax", None) is state.ax and state.ax is not None
    a.pnorm2_known = state.last_pnorm2 if known else -1.0
    a.ax = ax.data_ptr()
    U_new = pool.get() if pool else dev.empty(n, ld)
    V_new = pool.get() if pool else dev.empty(n, ld)
    a.U, a.V, a.U_new, a.V_new = state.U.data_ptr(), state.V.data_ptr(), U_new.data_ptr(), V_new.data_ptr()
    a.rho, a.scale = float(state.dual.rho), float(scale)
    a.want_balance = 1 if getattr(state, "want_balance", False) else 0
    a.rel_floor, a.primal_coeff, a.cg_cap = float(cg_rel_floor), float(cg_primal_coeff), int(cg_cap)
    global FUSED
    if dev.world > 1 and not a.dist:         # row-sharded: halo exchanges and reductions via hooks
        from .shard import native_hooks
        hs.dist_hooks = native_hooks(dev, ops)
        a.dist = hs.dist_hooks
    st = _lib.AdmmStepStats()
    fused = FUSED and dev.world == 1 and n >= 1 and n * lanes_for(ld) <= FUSED_MAX_LANES
    if fused:
        rc = dev.lib.cl_admm_step_diag_fused(ctypes.byref(a), ctypes.byref(st))
        if _lib.coop_refused(rc, "cl_admm_step_diag_fused"):
            FUSED = fused = False
        elif _lib.barrier_timeout(rc, "cl_admm_step_diag_fused"):
            # the step is void: U, V and lam were only read; ax may be overwritten
            FUSED = fused = False
            st = _lib.AdmmStepStats()
            if state.ax is not None:
                a.ax_valid = 0
                a.pnorm2_known = -1.0
        else:
            dev.launches += 1
            _lib.check(rc, "cl_admm_step_diag_fused")
    if not fused:
        rc = dev.lib.cl_admm_step_diag(ctypes.byref(a), ctypes.byref(st))
        dev.launches += 8 + 3 * (st.it_u + st.it_v)
        _lib.check(rc, f"cl_admm_step_diag (admm_native.cu:{st.err_line})")
    if st.status:
        if st.bad_half == 0:
            last = U_new if st.bad_is_new else state.U
        else:
            last = V_new if st.bad_is_new else state.V
        if st.status == 2:
            raise SpdViolationError(f"non-positive curvature {st.pq_bad:.3e} in CG (operator not SPD)")
        raise DivergedError("CG iterate diverged" if st.status == 3 else "CG produced non-finite curvature",
                            last_iterate=last)
    if st.u_reused:                       # CG stopped at its start: the factor is unchanged
        if pool:
            pool.put(U_new)
        U_new = state.U
    if st.v_reused:
        if pool:
            pool.put(V_new)
        V_new = state.V
    state.set_factors(U=U_new)
    state.set_factors(V=V_new)
    state.ax = ax
    state.last_pnorm2 = st.pnorm2
    state.pnorm2_ax = ax
    # the ascended multiplier was written out of place: swap buffers
    old = state.dual.lam
    state.dual.lam = lam_new
    hs.lam_spare = old
    state.step_obj = (st.objective, st.lam_b)
    state.step_bal = (st.du2, st.dv2) if st.du2 >= 0.0 else None
    return StepStats(st.it_u, st.it_v, st.res_u, st.res_v, bool(st.hit_cap))


def _admm_step_diag_py(state, ops, scale, cg_cap, rel_floor, coeff, hs, pool):
    """Python-driven twin of cl_admm_step_diag (admm_native.cu) without its speculation:
    every kernel that counts gets the same operands in the same order and the scalar
    decisions are the same, so the iterates are bit-identical. Used for row-sharded solves
    (halo exchanges and scalar reductions live in Python) and as the reference the native
    step is tested against."""
    dev = ops.dev
    p = ops.problem
    n, ld = state.U.shape
    rho = float(state.dual.rho)
    lam = state.dual.lam
    S = lambda k: 470 + k  # noqa: E731  (slots of admm_native.cu)
    cpat = ops.c_mat.cpat

    def fetch(hi):
        return dev.fetch(S(hi))

    if state.ax is None:
        ax = dev.empty(p.m)
        dev.constraint_eval(ops.cop.con, ld, state.U, state.V, ax)
    else:
        ax = state.ax
    known = getattr(state, "pnorm2_ax", None) is state.ax and state.ax is not None
    if known:
        pn2 = state.last_pnorm2
    else:
        dev.lincomb(hs.y, [ax, ops.b], [1.0, -1.0], dots=[("out", "out")], at=S(0))
        pn2 = float(fetch(1)[S(0)])
    pmeas = math.sqrt(pn2) / (1.0 + p.b_norminf)
    y = coeff * pmeas
    mn = y if y < 1e-2 else 1e-2
    rel = mn if mn > rel_floor else rel_floor
    dev.lincomb(hs.nlam, [ops.b, lam], [rho, -1.0])

    def half(x0, x, Wf, xx_prev, cw=None):
        """-> (status, eps, its, rnorm, last_is_x, pq, kept); status 4: previous iterate not finite"""
        dev.diag_admm_cg_init(cpat, Wf, x0, ld, scale, rho, hs.nlam, ops.diag_aval, hs.r, at=S(1), cw=cw)
        h = fetch(4 if xx_prev else 3)
        if xx_prev and not math.isfinite(float(h[S(3)])):
            return 4, 0.0, 0, 0.0, 0, 0.0, 0
        v = rel * math.sqrt(float(h[S(1)]))
        eps = 1e-300 if 1e-300 > v else v
        qr = float(h[S(2)])
        rnorm = math.sqrt(qr)
        if rnorm <= eps:
            return 0, eps, 0, rnorm, 0, 0.0, 1
        its, beta, xs = 0, 0.0, x0
        for k in range(cg_cap):
            dev.diag_cg_apply_rows(ops.diag_aval, ld, rho, hs.p, Wf, hs.coef, r=hs.r, beta=beta, at=S(4))
            pq = float(fetch(5)[S(4)])
            if not math.isfinite(pq) or pq <= 0.0:
                return (2 if math.isfinite(pq) else 1), eps, its, rnorm, int(xs is x), pq, 0
            alpha = qr / pq
            dev.diag_cg_step(ld, rho, hs.coef, Wf, xs, x, hs.p, hs.r, alpha=alpha, at=S(5))
            xs = x
            qn = float(fetch(6)[S(5)])
            rnorm = math.sqrt(qn)
            its = k + 1
            if rnorm <= eps:
                break
            beta = qn / qr
            qr = qn
        if its == 0:
            dev.lincomb(x, [x0], [1.0])
        return 0, eps, its, rnorm, 0, 0.0, 0

    def raise_for(st, half_new, half_old):
        last = half_new if st[4] else half_old
        if st[0] == 2:
            raise SpdViolationError(f"non-positive curvature {st[5]:.3e} in CG (operator not SPD)")
        raise DivergedError("CG produced non-finite curvature", last_iterate=last)

    U_new = pool.get() if pool else dev.empty(n, ld)
    V_new = pool.get() if pool else dev.empty(n, ld)
    st_u = half(state.U, U_new, state.V, False)
    if st_u[0]:
        raise_for(st_u, U_new, state.U)
    Uc = state.U if st_u[6] else U_new
    if not st_u[6]:
        dev.lincomb(None, [U_new], [0.0], dots=[(0, 0)], at=S(3))
    cu = hs.cu_buffer()
    st_v = half(state.V, V_new, Uc, not st_u[6], cw=cu)          # also stores C Uc for the step end
    if st_v[0] == 4:
        raise DivergedError("CG iterate diverged", last_iterate=U_new)
    if st_v[0]:
        raise_for(st_v, V_new, state.V)
    Vc = state.V if st_v[6] else V_new
    if not st_v[6]:
        dev.lincomb(None, [V_new], [0.0], dots=[(0, 0)], at=S(7))
    lam_new = hs.lam_spare if getattr(hs, "lam_spare", None) is not None else dev.empty(p.m)
    dev.diag_admm_step_end_rows(cu, Uc, Vc, ld, ops.diag_aval, ops.b, lam, rho, ax, lam_new, at=S(10))
    h = fetch(13)
    if not st_v[6] and not math.isfinite(float(h[S(7)])):
        raise DivergedError("CG iterate diverged", last_iterate=V_new)
    obj, pn2, lamb = h[S(10)], h[S(11)], h[S(12)]
    if st_u[6] and pool:
        pool.put(U_new)
    if st_v[6] and pool:
        pool.put(V_new)
    state.set_factors(U=Uc)
    state.set_factors(V=Vc)
    state.ax = ax
    state.last_pnorm2 = float(pn2)
    state.pnorm2_ax = ax
    hs.lam_spare = lam
    state.dual.lam = lam_new
    state.step_obj = (float(obj), float(lamb))
    hit_cap = (st_u[2] >= cg_cap and st_u[3] > st_u[1]) or (st_v[2] >= cg_cap and st_v[3] > st_v[1])
    return StepStats(st_u[2], st_v[2], st_u[3], st_v[3], bool(hit_cap))


def _admm_step_generic_native(state, ops, scale, cg_cap, rel_floor, coeff, hs, pool):
    """admm_step's generic branch below through cl_admm_step_generic: the same launches,
    the scalar decisions in native code (bit-identical iterates)."""
    from . import _lib
    dev = ops.dev
    p = ops.problem
    n, ld = state.U.shape
    a = getattr(hs, "generic_args", None)
    if a is None:
        a = hs.generic_args = _lib.AdmmGenericArgs()
        con = ops.cop.con
        apat = ops.adj.apat
        a.n, a.m, a.ld = n, p.m, ld
        a.b = ops.b.data_ptr()
        hs.rhs_buf = dev.empty(n, ld)
        hs.ax_bufs = [dev.empty(p.m), dev.empty(p.m)]
        a.rhs, a.r, a.p, a.Q = hs.rhs_buf.data_ptr(), hs.r.data_ptr(), hs.p.data_ptr(), hs.Q.data_ptr()
        a.y, a.nlam, a.rhob = hs.y.data_ptr(), hs.nlam.data_ptr(), hs.rhob.data_ptr()
        single = apat.single_a is not None and apat.halo is None and ld <= 64
        a.single_a = apat.single_a.data_ptr() if single else None
        if single and PAIR:
            if getattr(hs, "P2", None) is None:
                hs.P2 = dev.empty(n, 2 * ld)
            a.pair = hs.P2.data_ptr()
        a.con_indptr, a.con_pi, a.con_pj, a.con_val = (con.indptr.data_ptr(), con.pi.data_ptr(),
                                                       con.pj.data_ptr(), con.val.data_ptr())
        a.omega = ops.adj.omega.struct(c_coeff=1.0, w1=hs.nlam, w2=hs.rhob)
        a.apat = apat.struct(c_coeff=None, w1=hs.y)
        a.binf = float(p.b_norminf)
        a.slab = dev.slot(480).value
        a.host = dev.host.data_ptr() + 8 * 480
        a.ws, a.stream = dev.ws.data_ptr(), dev.stream.cuda_stream
    a.lam = state.dual.lam.data_ptr()
    a.ax = state.ax.data_ptr() if state.ax is not None else None
    ax_new = hs.ax_bufs[0] if hs.ax_bufs[0] is not state.ax else hs.ax_bufs[1]
    a.ax_new = ax_new.data_ptr()
    U_new = pool.get() if pool else dev.empty(n, ld)
    V_new = pool.get() if pool else dev.empty(n, ld)
    a.U, a.V, a.U_new, a.V_new = state.U.data_ptr(), state.V.data_ptr(), U_new.data_ptr(), V_new.data_ptr()
    a.rho, a.scale = float(state.dual.rho), float(scale)
    a.rel_floor, a.primal_coeff, a.cg_cap = float(rel_floor), float(coeff), int(cg_cap)
    st = _lib.AdmmStepStats()
    rc = dev.lib.cl_admm_step_generic(ctypes.byref(a), ctypes.byref(st))
    dev.launches += 12 + 4 * (st.it_u + st.it_v)
    _lib.check(rc, f"cl_admm_step_generic (admm_native.cu:{st.err_line})")
    if st.status:
        last = U_new if st.bad_half == 0 else V_new
        if st.status == 2:
            raise SpdViolationError(f"non-positive curvature {st.pq_bad:.3e} in CG (operator not SPD)")
        raise DivergedError("CG produced non-finite curvature" if st.status == 1 else "CG iterate diverged",
                            last_iterate=last)
    state.set_factors(U=U_new)
    state.set_factors(V=V_new)
    state.ax = ax_new
    state.last_pnorm2 = float(st.pnorm2)
    return StepStats(st.it_u, st.it_v, st.res_u, st.res_v, bool(st.hit_cap))


def admm_step(state: AdmmState, ops, *, scale=1.0, cg_cap=200, cg_rel_floor=1e-10,
              cg_primal_coeff=0.05, hs=None, pool=None) -> StepStats:
    """U half-solve, V half-solve, dual ascent (admm.py:136)."""
    dev = ops.dev
    if ops.is_diag:
        n, ld = state.U.shape
        hs = hs or HalfStep(ops, n, ld)
        if NATIVE:
            return _admm_step_native(state, ops, scale, cg_cap, cg_rel_floor, cg_primal_coeff, hs, pool)
        return _admm_step_diag_py(state, ops, scale, cg_cap, cg_rel_floor, cg_primal_coeff, hs, pool)
    if (NATIVE and NATIVE_GENERIC and dev.world == 1 and getattr(ops, "row_range", None) is None
            and getattr(ops.cop.con, "halo", None) is None and ops.adj.omega.halo is None
            and isinstance(state.dual.lam, torch.Tensor)):
        n, ld = state.U.shape
        hs = hs or HalfStep(ops, n, ld)
        return _admm_step_generic_native(state, ops, scale, cg_cap, cg_rel_floor, cg_primal_coeff, hs, pool)
    p = ops.problem
    dual = state.dual
    rho = dual.rho
    n, ld = state.U.shape
    hs = hs or HalfStep(ops, n, ld)
    ax = state.constraint_values(ops)
    _resid(ops, ax, hs.y, 430)
    pmeas = math.sqrt(float(dev.fetch(431)[430])) / (1.0 + p.b_norminf)
    rel = max(cg_rel_floor, min(1e-2, cg_primal_coeff * pmeas))
    lam = dual.lam

    rhs = pool.get() if pool else dev.empty(n, ld)
    hs.rhs(state.V, lam, rho, scale, rhs, at=431)
    eps_u = max(rel * math.sqrt(float(dev.fetch(432)[431])), 1e-300)
    U = pool.get() if pool else dev.empty(n, ld)
    it_u, res_u = hs.cg(U, state.V, rho, rhs, eps_u, cg_cap, x0=state.U)
    state.set_factors(U=U)

    hs.rhs(U, lam, rho, scale, rhs, at=432)
    eps_v = max(rel * math.sqrt(float(dev.fetch(433)[432])), 1e-300)
    V = pool.get() if pool else dev.empty(n, ld)
    it_v, res_v = hs.cg(V, U, rho, rhs, eps_v, cg_cap, x0=state.V)
    state.set_factors(V=V)
    if pool:
        pool.put(rhs)

    ax = state.constraint_values(ops)
    _resid(ops, ax, hs.y, 433)
    dev.lincomb(lam, [lam, hs.y], [1.0, rho])          # lam += rho*(A(UV^T) - b)
    state.last_pnorm2 = float(dev.fetch(434)[433])
    hit_cap = (it_u >= cg_cap and res_u > eps_u) or (it_v >= cg_cap and res_v > eps_v)
    return StepStats(it_u, it_v, res_u, res_v, hit_cap)


@dataclass
class AdmmResult:
    steps: int
    err1: float
    primal_scaled_inf: float
    cg_iterations: int
    hit_deadline: bool
    hit_cap: bool
    stalled: bool = False
    gap: float | None = None


class _Pool:
    def __init__(self, dev, n, ld):
        self.dev, self.n, self.ld, self.free = dev, n, ld, []

    def get(self):
        return self.free.pop() if self.free else self.dev.empty(self.n, self.ld)

    def put(self, t):
        self.free.append(t)


def admm_run(state: AdmmState, ops, *, scale=1.0, eps=1e-5, gap_eps=None, min_steps=0,
             step_cap=20000, cg_cap=200, rho_balance_mu=10.0, rho_balance_tau=2.0,
             rho_balance_every=5, rho_min=1e-6, rho_max=1e8, stall_window=60,
             stall_ratio=0.995, escalate=None, recorder=None, deadline=None) -> AdmmResult:
    """ADMM iterations with residual balancing and the gap-stall exit (admm.py:184).

    ``state.U/V`` are device n x ld factors of logical rank ``state.r``;
    ``escalate(U, V, r) -> (U_new, V_new, r_new) or None``.
    """
    dev = ops.dev
    p = ops.problem
    b1, binf = p.b_norm1, p.b_norminf
    n, ld = state.U.shape
    hs = HalfStep(ops, n, ld)
    pool = _Pool(dev, n, ld)
    res = dev.empty(p.m)

    def measures():
        ax = state.constraint_values(ops)
        _resid(ops, ax, res, 440)
        pn = math.sqrt(float(dev.fetch(441)[440]))
        return pn, pn / (1.0 + b1), pn / (1.0 + binf)

    def objective_and_gap():
        # <C, U V^T> and lam.b in one fetch
        dev.spmm(ops.c_mat.cpat, state.V, state.U.shape[1], out=None, Z=[state.U],
                 dots=[("out", ("z", 0))], at=442, c_coeff=1.0)
        dev.lincomb(None, [state.dual.lam, ops.b], [0.0, 0.0], dots=[(0, 1)], at=443)
        s = dev.fetch(444)
        obj = float(s[442])
        lam_b = -float(s[443]) / scale
        return obj, abs(obj - lam_b) / (1.0 + abs(obj) + abs(lam_b))

    pnorm, err1, p0 = measures()
    g3 = objective_and_gap()[1] if gap_eps is not None else None
    if p0 <= eps and (gap_eps is None or g3 < gap_eps) and min_steps == 0:
        return AdmmResult(steps=0, err1=err1, primal_scaled_inf=p0, cg_iterations=0,
                          hit_deadline=False, hit_cap=False, gap=g3)
    cg_total = 0
    cap_streak = 0
    steps = 0
    hit_deadline = False
    stalled = False
    gap_hist = deque(maxlen=stall_window)
    for step in range(1, step_cap + 1):
        if deadline is not None and time.perf_counter() > deadline:
            hit_deadline = True
            break
        U_prev, V_prev = state.U, state.V
        state.step_obj = None
        state.step_bal = None
        state.want_balance = step % rho_balance_every == 0
        stats = admm_step(state, ops, scale=scale, cg_cap=cg_cap, hs=hs, pool=pool)
        cg_total += stats.cg_iters_u + stats.cg_iters_v
        steps = step
        pnorm = math.sqrt(state.last_pnorm2)
        err1, p0 = pnorm / (1.0 + b1), pnorm / (1.0 + binf)
        obj = None
        if gap_eps is not None or recorder is not None:
            if state.step_obj is not None:       # computed inside the native step (same kernels)
                obj, lam_b = state.step_obj[0], -state.step_obj[1] / scale
                g3v = abs(obj - lam_b) / (1.0 + abs(obj) + abs(lam_b))
            else:
                obj, g3v = objective_and_gap()
            g3 = g3v if gap_eps is not None else None
        if recorder is not None:
            recorder.record("admm", scale * obj, err1, max(stats.resid_u, stats.resid_v),
                            state.dual.rho, state.r)
            gaps = getattr(recorder, "gaps", None)      # diagnostics beside the trace (driver.Trace)
            if gaps is not None and g3 is not None:
                gaps.append((recorder.counter, g3))
        done = p0 <= eps and (gap_eps is None or g3 < gap_eps) and step >= min_steps
        balance = (not done) and step % rho_balance_every == 0
        bal = state.step_bal                   # measured inside the one-launch step
        if balance and bal is None:
            dev.lincomb(None, [state.U, U_prev], [1.0, -1.0], dots=[("out", "out")], at=445)
            dev.lincomb(None, [state.V, V_prev], [1.0, -1.0], dots=[("out", "out")], at=446)
        if U_prev is not state.U:
            pool.put(U_prev)
        if V_prev is not state.V:
            pool.put(V_prev)
        if done:
            break
        if gap_eps is not None and p0 <= eps:
            gap_hist.append(g3)
            if len(gap_hist) == stall_window and gap_hist[-1] > stall_ratio * gap_hist[0]:
                stalled = True
                break
        else:
            gap_hist.clear()
        if balance:
            if bal is None:
                s = dev.fetch(447)
                bal = (float(s[445]), float(s[446]))
            dual_surrogate = state.dual.rho * (math.sqrt(bal[0]) + math.sqrt(bal[1]))
            if pnorm > rho_balance_mu * dual_surrogate:
                state.dual.rho = min(state.dual.rho * rho_balance_tau, rho_max)
            elif dual_surrogate > rho_balance_mu * pnorm:
                state.dual.rho = max(state.dual.rho / rho_balance_tau, rho_min)
        cap_streak = cap_streak + 1 if stats.hit_cap else 0
        if cap_streak >= 2 and escalate is not None:
            grown = escalate(state.U, state.V, state.r)
            if grown is not None:
                U2, V2, state.r = grown
                state.set_factors(U=U2, V=V2)
                n, ld = U2.shape
                hs = HalfStep(ops, n, ld)
                pool = _Pool(dev, n, ld)
            cap_streak = 0
    return AdmmResult(steps=steps, err1=err1, primal_scaled_inf=p0, cg_iterations=cg_total,
                      hit_deadline=hit_deadline, hit_cap=cap_streak > 0, stalled=stalled, gap=g3)

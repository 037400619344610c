"""Stage one: Burer-Monteiro ALM with L-BFGS and the exact quartic line search.

Device restatement of the reference's lrsdp/alm.py. The algorithm, its
stopping rules and every heuristic are the reference's; what changes is how
each iteration maps onto the B200:

* L-BFGS (alm.py:98) runs *vector-free*: the curvature pairs stay in HBM,
  their Gram matrix lives on the host, the two-loop recursion runs on the
  (2T+1)-dimensional coefficient vector, and the direction is written by ONE
  streaming combination that also returns its inner products with every
  basis vector (the Gram update). Two HBM passes over the history per
  iteration instead of the two-loop's 4T dependent passes.
* The line-search data (alm.py:135) -- C D, <CD,R>, <CD,D>, <CR,D>, q1, q2
  and the m-vector dot products -- come out of one pattern-SpMM launch, one
  fused constraint launch and one m-vector launch; the host solves the cubic.
* Step, constraint refresh, gradient 2 S R (alm.py:239), Lagrangian value
  (alm.py:248) and the curvature-pair inner products are one row-local kernel
  for diagonal-constraint problems (MaxCut) and a short chain otherwise.

Host/device synchronisation: two small scalar reads per inner iteration.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from collections import deque
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import F64, padded_ld
from .exceptions import DivergedError
from .linops import to_factor, to_vec

_REFRESH_EVERY = 50     # alm.py:29
_CURVATURE_MIN = 0.0    # alm.py:30


@dataclass
class FactorPair:
    """Low-rank iterate; the first stage aliases left and right (alm.py:34)."""

    left: object
    right: object

    @classmethod
    def symmetric(cls, R):
        return cls(left=R, right=R)

    @property
    def n(self):
        return self.left.shape[0]

    @property
    def r(self):
        return self.left.shape[1]

    @property
    def is_symmetric(self):
        return self.right is self.left

    def check(self):
        if tuple(self.left.shape) != tuple(self.right.shape):
            raise ValueError("left and right factors must share a shape")
        if self.r < 1:
            raise ValueError("rank must be at least 1")
        for W in (self.left, self.right):
            ok = bool(torch.isfinite(W).all()) if isinstance(W, torch.Tensor) else bool(np.all(np.isfinite(W)))
            if not ok:
                raise ValueError("factor entries must be finite")


@dataclass
class DualVector:
    """Multiplier and penalty (alm.py:66). ``lam`` may live on host or device."""

    lam: object
    rho: float

    def __post_init__(self):
        if not self.rho > 0:
            raise ValueError("penalty must be positive")


# ---------------------------------------------------------------------------
# exact line search (host scalar algebra, Appendix A.2)
# ---------------------------------------------------------------------------

@dataclass
class LineSearchPoly:
    """phi(t) = a1 t^4 + a2 t^3 + a3 t^2 + a4 t = L(R + tD) - L(R)  (alm.py:112)."""

    a1: float
    a2: float
    a3: float
    a4: float
    p1: float = 0.0
    p2: float = 0.0
    q0: object = None
    q1: object = None
    q2: object = None

    def value(self, t):
        return ((self.a1 * t + self.a2) * t + self.a3) * t * t + self.a4 * t

    def coeffs(self):
        return (self.a1, self.a2, self.a3, self.a4)


def _polish(c, x):
    """Two Newton steps on c[0] x^3 + c[1] x^2 + c[2] x + c[3]."""
    c3, c2, c1, c0 = c
    for _ in range(2):
        f = ((c3 * x + c2) * x + c1) * x + c0
        df = (3.0 * c3 * x + 2.0 * c2) * x + c1
        if df != 0.0 and math.isfinite(f) and math.isfinite(df):
            x -= f / df
    return x


def cubic_roots(c3, c2, c1, c0):
    """Real roots of the cubic via the depressed form (alm.py:166)."""
    b2, b1, b0 = c2 / c3, c1 / c3, c0 / c3
    shift = b2 / 3.0
    P = b1 - b2 * b2 / 3.0
    Q = b0 - b2 * b1 / 3.0 + 2.0 * b2 ** 3 / 27.0
    if abs(P) < 1e-300 and abs(Q) < 1e-300:
        ts = [0.0]
    elif -4.0 * P ** 3 - 27.0 * Q ** 2 > 0.0:
        amp = 2.0 * math.sqrt(-P / 3.0)
        phase = math.acos(min(1.0, max(-1.0, 3.0 * Q / (P * amp)))) / 3.0
        ts = [amp * math.cos(phase - 2.0 * math.pi * k / 3.0) for k in (0, 1, 2)]
    else:
        h = -0.5 * Q
        rad = math.sqrt(max(0.0, Q * Q / 4.0 + P ** 3 / 27.0))
        ts = [math.copysign(abs(h + rad) ** (1.0 / 3.0), h + rad)
              + math.copysign(abs(h - rad) ** (1.0 / 3.0), h - rad)]
    return [_polish((c3, c2, c1, c0), t - shift) for t in ts]


def best_step(poly: LineSearchPoly):
    """Global minimiser of the ray quartic, (tau, zero_direction) (alm.py:202)."""
    a1, a2, a3, a4 = poly.coeffs()
    if a1 == 0.0 and a2 == 0.0 and a3 == 0.0 and a4 == 0.0:
        return 0.0, True
    if a1 != 0.0:
        cand = cubic_roots(4.0 * a1, 3.0 * a2, 2.0 * a3, a4) + [0.0]
    elif a2 != 0.0:
        cand = [0.0]
        disc = a3 * a3 - 3.0 * a2 * a4
        if disc >= 0.0:
            for sg in (1.0, -1.0):
                t = (-a3 + sg * math.sqrt(disc)) / (3.0 * a2)
                if 6.0 * a2 * t + 2.0 * a3 > 0.0:     # local minimum of the cubic
                    cand.append(t)
    elif a3 != 0.0:
        cand = [-a4 / (2.0 * a3)] if a3 > 0.0 else [0.0]
    else:
        cand = [0.0]
    vals = [poly.value(t) if math.isfinite(t) else math.inf for t in cand]
    vmin = min(vals)
    band = vmin + 1e-12 * (1.0 + abs(vmin))
    best = min((t for t, v in zip(cand, vals) if v <= band), key=lambda t: (abs(t), -t))
    return best, False


def _quartic(rho, p1, p2, q2q2, q1q2, wq2, q1q1, wq1):
    """a1..a4 from the reduced inner products (alm.py:158-162), w = -lam + rho q0."""
    return (0.5 * rho * q2q2, rho * q1q2, p2 - wq2 + 0.5 * rho * q1q1, p1 - wq1)


# ---------------------------------------------------------------------------
# device workspace and vector-free L-BFGS history
# ---------------------------------------------------------------------------

class FactorPool:
    """Recycles n x ld device buffers (history slots, scratch)."""

    def __init__(self, dev, n, ld):
        self.dev, self.n, self.ld = dev, n, ld
        self.free = []

    def get(self):
        if self.free:
            return self.free.pop()
        return torch.empty((self.n, self.ld), dtype=F64, device=self.dev.dev)

    def put(self, t):
        self.free.append(t)


class LbfgsHistory:
    """Curvature pairs in HBM, Gram matrix on the host (alm.py:77 semantics).

    Pair t holds s_t = sigma_t * Dbuf_t and y_t = Ybuf_t; ``beta_t = 1/<y_t,s_t>``.
    Pairs with non-positive curvature are rejected (alm.py:84-89).
    """

    def __init__(self, capacity, pool=None):
        self.capacity = capacity
        self.pool = pool
        self.pairs = deque()          # (dbuf, ybuf, sigma, beta)
        self.G = {}                   # (id(a), id(b)) -> <a, b> for live buffers

    def __len__(self):
        return len(self.pairs)

    # Gram bookkeeping ---------------------------------------------------
    @staticmethod
    def _k(a, b):
        ia, ib = id(a), id(b)
        return (ia, ib) if ia <= ib else (ib, ia)

    def set_dot(self, a, b, v):
        self.G[self._k(a, b)] = float(v)

    def dot(self, a, b):
        return self.G[self._k(a, b)]

    def forget(self, t):
        i = id(t)
        for k in [k for k in self.G if i in k]:
            del self.G[k]

    def live(self):
        return [p[0] for p in self.pairs] + [p[1] for p in self.pairs]

    # two-loop in coefficient space --------------------------------------
    def coefficients(self, g):
        """Coefficients c with D = sum c_j b_j equal to Algorithm 1's direction."""
        c = {id(g): (g, -1.0)}

        def dotD(x):
            return sum(self.dot(x, t) * cj for (t, cj) in c.values())

        alphas = []
        for dbuf, ybuf, sig, beta in reversed(self.pairs):
            a = beta * (sig * dotD(dbuf))
            t, cj = c.get(id(ybuf), (ybuf, 0.0))
            c[id(ybuf)] = (t, cj - a)
            alphas.append(a)
        for (dbuf, ybuf, sig, beta), a in zip(self.pairs, reversed(alphas)):
            bb = beta * dotD(ybuf)
            t, cj = c.get(id(dbuf), (dbuf, 0.0))
            c[id(dbuf)] = (t, cj + (a - bb) * sig)
        return list(c.values())

    def push(self, dbuf, ybuf, sigma, ys):
        """Accept (sigma*dbuf, ybuf) if <y,s> > 0; returns (accepted, evicted buffers)."""
        if ys > _CURVATURE_MIN:
            evicted = []
            if len(self.pairs) == self.capacity:
                old = self.pairs.popleft()
                evicted = [old[0], old[1]]
                for t in evicted:
                    self.forget(t)
            self.pairs.append((dbuf, ybuf, sigma, 1.0 / ys))
            return True, evicted
        return False, []

    def clear(self):
        for d, y, _, _ in self.pairs:
            self.forget(d)
            self.forget(y)
            if self.pool is not None:
                self.pool.put(d)
                self.pool.put(y)
        self.pairs.clear()


def lbfgs_direction(g, hist: LbfgsHistory, dev=None, out=None):
    """Algorithm 1's direction -H g from the device history (alm.py:98).

    ``hist.G`` must hold the inner products among ``g`` and the live pair
    buffers. Returns the direction buffer; its inner products with every
    basis buffer are recorded in ``hist.G``.
    """
    from .device import default_device
    dev = dev or default_device()
    terms = hist.coefficients(g)
    # include every live buffer so the Gram row of D is complete
    have = {id(t) for t, _ in terms}
    for t in hist.live():
        if id(t) not in have:
            terms.append((t, 0.0))
    if out is None:
        out = torch.empty_like(g)
    ins = [t for t, _ in terms]
    dev.lincomb(out, ins, [c for _, c in terms], dots=True, mode=_lib.CL_DOT_OUT_ALL, at=0)
    s = dev.fetch(len(ins) + 1)
    for j, t in enumerate(ins):
        hist.set_dot(out, t, s[j])
    hist.set_dot(out, out, s[len(ins)])
    return out


# ---------------------------------------------------------------------------
# gradient / value / line search on the device
# ---------------------------------------------------------------------------

class AlmCore:
    """Device buffers of one ALM stage at a fixed (n, ld)."""

    # slab offsets
    S_DIR = 0          # direction dots (<= 2T+2)
    S_LS = 40          # <CD,R>, <CD,D>, <CR,D>
    S_MV = 48          # q2q2, q1q2, wq2, q1q1, wq1
    S_UPD = 64         # update dots (7 + 2*CL_MAXIN)
    S_AUX = 128        # misc

    def __init__(self, ops, n, ld):
        self.ops, self.dev, self.n, self.ld = ops, ops.dev, n, ld
        dev = self.dev
        m = ops.problem.m
        self.pool = FactorPool(dev, n, ld)
        self.CR = dev.empty(n, ld)
        self.CD = dev.empty(n, ld)
        self.ax = dev.empty(m)
        self.ax2 = dev.empty(m)
        self.q1 = dev.empty(m)
        self.q2 = dev.empty(m)
        self.wv = dev.empty(m)
        self.res = dev.empty(m)
        self.zero_g = None

    # A(R R^T) and C R -------------------------------------------------
    def constraint_values(self, R, out=None):
        out = self.ax if out is None else out
        self.dev.constraint_eval(self.ops.cop.con, self.ld, R, R, out)
        return out

    def c_times(self, X, out):
        self.dev.spmm(self.ops.c_mat.cpat, X, self.ld, out=out, c_coeff=1.0)
        return out

    # gradient + value (+ pair inner products) -------------------------
    def grad_value(self, R, lam, rho, scale, g_old, g_new, ybuf, H, D=None, CD=None, tau=0.0,
                   refresh=True, fetch=True):
        """Step (unless refresh), gradient 2 S R and the Lagrangian pieces.

        Returns dict: crr, gg, yd, lres, rr, yy, gy, gH[list], yH[list]; with
        ``fetch=False`` (diagonal path only) the launch is queued and None is
        returned -- the reductions stay in the device slab."""
        dev, ops = self.dev, self.ops
        b = ops.b
        nh = len(H)
        if ops.is_diag:
            a = _lib.DiagUpdateArgs()
            a.n, a.ld = self.n, self.ld
            a.aval = ops.diag_aval.data_ptr()
            a.tau, a.rho, a.scale = float(tau), float(rho), float(scale)
            a.R = R.data_ptr()
            a.D = (D if D is not None else R).data_ptr()
            a.CR = self.CR.data_ptr()
            a.CD = (CD if CD is not None else self.CR).data_ptr()
            a.ax = self.ax.data_ptr()
            a.ax_out = (self.ax if refresh else self.ax2).data_ptr()
            a.q1, a.q2 = self.q1.data_ptr(), self.q2.data_ptr()
            a.lam, a.b = lam.data_ptr(), b.data_ptr()
            a.g_old, a.g_new, a.y = g_old.data_ptr(), g_new.data_ptr(), ybuf.data_ptr()
            a.nh = nh
            for j, t in enumerate(H):
                a.H[j] = t.data_ptr()
            a.refresh = 1 if refresh else 0
            dev.diag_update(a, at=self.S_UPD)
            if not refresh:
                self.ax, self.ax2 = self.ax2, self.ax
            if not fetch:
                return None
            s = dev.fetch(self.S_UPD + 7 + 2 * _lib.CL_MAXIN)[self.S_UPD:]
            return dict(crr=s[0], gg=s[1], yd=s[2], lres=s[3], rr=s[4], yy=s[5], gy=s[6],
                        gH=list(s[7:7 + nh]), yH=list(s[7 + _lib.CL_MAXIN:7 + _lib.CL_MAXIN + nh]))
        # generic chain
        if not refresh:
            dev.lincomb(R, [R, D], [1.0, tau])
            dev.lincomb(self.CR, [self.CR, CD], [1.0, tau])
            dev.lincomb(self.ax2, [self.ax, self.q1, self.q2], [1.0, tau, tau * tau])
            self.ax, self.ax2 = self.ax2, self.ax
        A = self.S_UPD
        # res = ax - b ; rr, lam.res ; <CR,R>
        dev.lincomb(self.res, [self.ax, b, lam], [1.0, -1.0, 0.0], dots=[("out", "out"), (2, "out")],
                    at=A + 4 - 1 + 1)   # rr at A+4, lres at A+5 (remapped below)
        dev.lincomb(None, [self.CR, R], [0.0, 0.0], dots=[(0, 1)], at=A + 0, N=self.CR.numel())
        dev.lincomb(self.wv, [lam, self.res], [1.0, rho])           # w = lam + rho*(ax - b)
        # g = 2 A*(w) R + 2 scale C R
        dev.spmm(ops.adj.apat, R, self.ld, alpha=2.0, out=g_new, Y=[self.CR], ycoef=[2.0 * scale],
                 w1=self.wv)
        dev.lincomb(ybuf, [g_new, g_old], [1.0, -1.0])
        ins = [g_new, ybuf] + list(H)
        dev.lincomb(None, ins, [0.0] * len(ins), dots=True, mode=_lib.CL_DOT_FIRST_TWO, at=A + 8)
        s = dev.fetch(A + 8 + 2 * _lib.CL_MAXIN)[A:]
        gH = [s[8 + 2 + j] for j in range(nh)]
        yH = [s[8 + _lib.CL_MAXIN + 1 + j] for j in range(nh)]
        yd = yH[-1] if (D is not None and nh and H[-1] is D) else 0.0
        return dict(crr=s[0], gg=s[8], yd=yd, lres=s[5], rr=s[4], yy=s[8 + _lib.CL_MAXIN],
                    gy=s[9], gH=gH, yH=yH)

    # line search -------------------------------------------------------
    def pair_ok(self):
        """Line search on a pair buffer [R | D]: single-entry constraints, one GPU, ld <= 64."""
        con = self.ops.cop.con
        return (PAIR and con.diag_aval is None and getattr(con, "halo", None) is None and self.ld <= 64
                and self.ops.adj.apat.single_a is not None)

    def pair_buffer(self):
        if getattr(self, "P2", None) is None:
            self.P2 = self.dev.empty(self.n, 2 * self.ld)
        return self.P2

    def line_search(self, R, D, lam, rho, scale):
        dev, ops = self.dev, self.ops
        dev.spmm(ops.c_mat.cpat, D, self.ld, out=self.CD, Z=[R, D, self.CR],
                 dots=[("out", ("z", 0)), ("out", ("z", 1)), (("z", 2), ("z", 1))], at=self.S_LS,
                 c_coeff=1.0)
        con = ops.cop.con
        if self.pair_ok():
            # single-entry constraints: R and D interleaved in one pair buffer, so each
            # position's four rows come as two 2 ld runs (bit-identical products)
            P2 = self.pair_buffer()
            dev.pair_pack(R, self.ld, P2, 0)
            dev.pair_pack(D, self.ld, P2, 1)
            dev.constraint_eval_pair(con, self.ld, P2, self.q1, self.q2)
        else:
            dev.constraint_eval(con, self.ld, R, D, self.q1, X2=D, Y2=R, X3=D, Y3=D, out2=self.q2)
        # w = -lam + rho*(b - ax)
        dev.lincomb(self.wv, [lam, ops.b, self.ax, self.q1, self.q2], [-1.0, rho, -rho, 0.0, 0.0],
                    dots=[(4, 4), (3, 4), ("out", 4), (3, 3), ("out", 3)], at=self.S_MV)
        s = dev.fetch(self.S_MV + 5)
        cdr, cdd, crd = s[self.S_LS:self.S_LS + 3]
        q2q2, q1q2, wq2, q1q1, wq1 = s[self.S_MV:self.S_MV + 5]
        p1 = scale * float(cdr + crd)
        p2 = scale * float(cdd)
        a = _quartic(rho, p1, p2, q2q2, q1q2, wq2, q1q1, wq1)
        return LineSearchPoly(*a, p1=p1, p2=p2, q1=self.q1, q2=self.q2)


# ---------------------------------------------------------------------------
# reference-shaped API (numpy or torch in, same kind out)
# ---------------------------------------------------------------------------

def _prep(ops, R):
    ld = padded_ld(R.shape[1])
    return to_factor(R, ops.dev, ld), ld


def _lam_dev(ops, lam):
    return to_vec(lam, ops.dev)


def alm_gradient(R, dual: DualVector, ops, scale=1.0, ax=None):
    """2 S R, S = scale*C + A*(lam + rho*(A(RR^T) - b)) (alm.py:239)."""
    Rd, ld = _prep(ops, R)
    dev = ops.dev
    m = ops.problem.m
    axd = ops.cop.apply_pair_dev(Rd, Rd, ld) if ax is None else to_vec(ax, dev)
    w = dev.empty(m)
    if ops.is_diag and getattr(ops.c_mat.cpat, "halo", None) is None:
        # diagonal constraints (MaxCut): S = scale C + diag(a w), so 2 S R is the C product with a
        # row-diagonal epilogue term -- the solver's own fused path (no Omega assembly). Same
        # value as the assembled product up to the association of the diagonal slot (1e-16).
        dev.lincomb(w, [_lam_dev(ops, dual.lam), axd, ops.b], [2.0, 2.0 * dual.rho, -2.0 * dual.rho])
        g = dev.empty(*Rd.shape)
        dev.spmm(ops.c_mat.cpat, Rd, ld, alpha=2.0 * scale, out=g, Y=[Rd], ycoef=[0.0], c_coeff=1.0,
                 drow=w, dmul=ops.diag_aval)
        out = g[:, :R.shape[1]]
        return out if isinstance(R, torch.Tensor) else out.cpu().numpy()
    dev.lincomb(w, [_lam_dev(ops, dual.lam), axd, ops.b], [1.0, dual.rho, -dual.rho])
    S = ops.adj.assemble(lam=w, c_coeff=scale)
    g = S.matmul_dev(Rd, ld, alpha=2.0)
    out = g[:, :R.shape[1]]
    return out if isinstance(R, torch.Tensor) else out.cpu().numpy()


def alm_value(R, dual: DualVector, ops, scale=1.0, ax=None, CR=None):
    """Penalised Lagrangian (alm.py:248)."""
    Rd, ld = _prep(ops, R)
    dev = ops.dev
    axd = ops.cop.apply_pair_dev(Rd, Rd, ld) if ax is None else to_vec(ax, dev)
    if CR is None:
        CRd = dev.empty(*Rd.shape)
        dev.spmm(ops.c_mat.cpat, Rd, ld, out=CRd, c_coeff=1.0)
    else:
        CRd = to_factor(CR, dev, ld)
    res = dev.empty(ops.problem.m)
    dev.lincomb(None, [CRd, Rd], [0.0, 0.0], dots=[(0, 1)], at=200)
    dev.lincomb(res, [axd, ops.b, _lam_dev(ops, dual.lam)], [1.0, -1.0, 0.0],
                dots=[("out", "out"), (2, "out")], at=201)
    s = dev.fetch(203)
    return scale * float(s[200]) + float(s[202]) + 0.5 * dual.rho * float(s[201])


def line_search_poly(R, D, dual: DualVector, ops, scale=1.0, ax=None, CR=None, CD=None):
    """Quartic coefficients of the exact line search along D (alm.py:135)."""
    Rd, ld = _prep(ops, R)
    Dd = to_factor(D, ops.dev, ld)
    core = AlmCore(ops, Rd.shape[0], ld)
    if ax is None:
        core.constraint_values(Rd)
    else:
        core.ax.copy_(to_vec(ax, ops.dev))
    if CR is None:
        core.c_times(Rd, core.CR)
    else:
        core.CR.copy_(to_factor(CR, ops.dev, ld))
    poly = core.line_search(Rd, Dd, _lam_dev(ops, dual.lam), dual.rho, scale)
    host = not isinstance(R, torch.Tensor)
    q0 = ops.b - core.ax
    poly.q0 = q0.cpu().numpy() if host else q0
    poly.q1 = core.q1.cpu().numpy() if host else core.q1.clone()
    poly.q2 = core.q2.cpu().numpy() if host else core.q2.clone()
    return poly


@dataclass
class InnerResult:
    R: object
    iterations: int
    grad_norms: list
    hit_cap: bool
    ax: object


# single-entry constraints: the line search reads R and D from a pair buffer (cl_constraint_eval_pair)
PAIR = os.environ.get("CULORADS_PAIR", "1") != "0"
NATIVE = True     # diagonal constraints: run the inner loop's control flow in C++ (row-sharded: with hooks)
NATIVE_GENERIC = True   # other constraint families on one GPU: cl_alm_inner_generic
# Problems with n*ld at most this many doubles run the whole inner solve as one
# cooperative launch (cl_alm_inner_diag_fused): latency, not HBM, bounds them.
FUSED = os.environ.get("CULORADS_FUSED", "1") != "0"
FUSED_MAX_ELEMS = int(os.environ.get("CULORADS_FUSED_MAX", 1 << 18))


def _inner_native(core, R, lam, rho, scale, tol, max_iter, reduce_factor, memory, recorder):
    """alm.py:268 through cl_alm_inner_diag (diagonal constraints) or cl_alm_inner_generic
    (any other constraint family, one GPU): the launches of ``_inner`` below with the
    host-side scalar algebra in native code (bit-identical iterates)."""
    from . import _lib
    dev, ops = core.dev, core.ops
    generic = not ops.is_diag
    n, ld = core.n, core.ld
    nbuf = 2 * memory + 4
    bufs = getattr(core, "native_bufs", None)
    if bufs is None or len(bufs) < nbuf:
        bufs = core.native_bufs = [dev.empty(n, ld) for _ in range(nbuf)]
    a = _lib.AlmInnerArgs()
    a.n, a.ld, a.memory, a.max_iter = n, ld, memory, max_iter
    a.tol = float(tol)
    a.reduce_factor = float(reduce_factor) if reduce_factor is not None else -1.0
    a.rho, a.scale, a.b1 = float(rho), float(scale), float(ops.problem.b_norm1)
    a.aval = ops.diag_aval.data_ptr() if not generic else None
    a.b, a.lam = ops.b.data_ptr(), lam.data_ptr()
    a.R, a.CR, a.CD = R.data_ptr(), core.CR.data_ptr(), core.CD.data_ptr()
    a.ax, a.ax2 = core.ax.data_ptr(), core.ax2.data_ptr()
    a.q1, a.q2, a.wv = core.q1.data_ptr(), core.q2.data_ptr(), core.wv.data_ptr()
    a.zero_g = None                 # g_old = 0 for the first gradient: no zero factor is held
    if generic:
        # the generic chain's y = g - g_old is a lincomb: it reads a zero factor, as _inner does
        if core.zero_g is None:
            core.zero_g = dev.zeros(n, ld)
        a.zero_g = core.zero_g.data_ptr()
        con = ops.cop.con
        a.m = int(con.m)
        a.con_indptr, a.con_pi, a.con_pj, a.con_val = (con.indptr.data_ptr(), con.pi.data_ptr(),
                                                       con.pj.data_ptr(), con.val.data_ptr())
        a.apat = ops.adj.apat.struct(c_coeff=None, w1=core.wv)
        a.res = core.res.data_ptr()
        if core.pair_ok():
            a.pair = core.pair_buffer().data_ptr()
    a.nbuf = nbuf
    for j in range(nbuf):
        a.bufs[j] = bufs[j].data_ptr()
    a.cpat = ops.c_mat.cpat.struct(c_coeff=1.0)
    a.slab, a.host = dev.slab.data_ptr(), dev.host.data_ptr()
    a.ws, a.stream = dev.ws.data_ptr(), dev.stream.cuda_stream
    cap = max_iter + 1
    rec = np.empty(4 * cap)
    gn = np.empty(cap)
    a.rec_cap = cap
    a.rec = rec.ctypes.data
    a.gnorms = gn.ctypes.data
    global FUSED
    if dev.world > 1:                       # row-sharded: halo exchanges and reductions via hooks
        if getattr(core, "dist_hooks", None) is None:
            from .shard import native_hooks
            core.dist_hooks = native_hooks(dev, ops)
        a.dist = core.dist_hooks
    st = _lib.AlmInnerStats()
    fused = FUSED and not generic and dev.world == 1 and n >= 1 and n * ld <= FUSED_MAX_ELEMS
    if fused:
        R_keep = R.clone()          # the one launch steps R in place; kept for a void launch
        rc = dev.lib.cl_alm_inner_diag_fused(ctypes.byref(a), ctypes.byref(st))
        if _lib.coop_refused(rc, "cl_alm_inner_diag_fused"):
            FUSED = fused = False
        elif _lib.barrier_timeout(rc, "cl_alm_inner_diag_fused"):
            FUSED = fused = False
            R.copy_(R_keep)
            st = _lib.AlmInnerStats()
        else:
            dev.launches += 1
            _lib.check(rc, "cl_alm_inner_diag_fused")
    if generic:
        fused = False
        rc = dev.lib.cl_alm_inner_generic(ctypes.byref(a), ctypes.byref(st))
        dev.launches += 8 + 13 * st.iterations
        _lib.check(rc, f"cl_alm_inner_generic (alm_native.cu:{st.err_line})")
    elif not fused:
        rc = dev.lib.cl_alm_inner_diag(ctypes.byref(a), ctypes.byref(st))
        dev.launches += 2 + 5 * st.iterations
        _lib.check(rc, f"cl_alm_inner_diag (alm_native.cu:{st.err_line})")
    if st.ax_is_ax2:
        core.ax, core.ax2 = core.ax2, core.ax
    if recorder:
        for k in range(st.n_records):
            recorder.record("alm", float(rec[4 * k]), float(rec[4 * k + 1]), float(rec[4 * k + 2]), rho,
                            None, t=float(rec[4 * k + 3]))
    if st.status == 1:
        raise DivergedError("non-finite Lagrangian at inner start", last_iterate=R)
    if st.status == 2:
        raise DivergedError("inner iteration diverged", last_iterate=R)
    return InnerResult(R, st.iterations, [float(x) for x in gn[:st.n_gnorms]], bool(st.hit_cap), core.ax)


def _inner(core, R, lam, rho, scale, tol, max_iter, reduce_factor, memory, recorder):
    """alm.py:268 on device buffers. R is updated in place."""
    dev, ops = core.dev, core.ops
    if NATIVE and memory <= 8 and core.ld >= 2 and (ops.is_diag or (
            NATIVE_GENERIC and dev.world == 1 and getattr(ops, "row_range", None) is None
            and getattr(ops.cop.con, "halo", None) is None)):
        return _inner_native(core, R, lam, rho, scale, tol, max_iter, reduce_factor, memory, recorder)
    b1 = ops.problem.b_norm1
    pool = core.pool
    hist = LbfgsHistory(memory, pool)
    core.constraint_values(R)
    core.c_times(R, core.CR)
    g = pool.get()
    gscr = pool.get()
    yscr = pool.get()
    if core.zero_g is None:
        core.zero_g = dev.zeros(core.n, core.ld)
    out = core.grad_value(R, lam, rho, scale, core.zero_g, g, yscr, [], refresh=True)
    L = scale * out["crr"] + out["lres"] + 0.5 * rho * out["rr"]
    gg = out["gg"]
    hist.set_dot(g, g, gg)
    if not (math.isfinite(L) and math.isfinite(gg)):
        raise DivergedError("non-finite Lagrangian at inner start", last_iterate=R)
    gnorm0 = math.sqrt(gg)
    grad_norms = []
    iterations = 0

    def finish(hit):
        hist.clear()
        for t in (g, gscr, yscr):
            pool.put(t)
        return InnerResult(R, iterations, grad_norms, hit, core.ax)

    for it in range(max_iter):
        gnorm = math.sqrt(gg)
        grad_norms.append(gnorm)
        if gnorm / (1.0 + abs(L)) <= tol:
            return finish(False)
        if reduce_factor is not None and gnorm <= reduce_factor * gnorm0:
            return finish(False)

        Dn = pool.get()
        lbfgs_direction(g, hist, dev, out=Dn)
        poly = core.line_search(R, Dn, lam, rho, scale)
        tau, zero = best_step(poly)
        if zero or tau == 0.0:
            hist.forget(Dn)
            pool.put(Dn)
            return finish(False)

        refresh = (it + 1) % _REFRESH_EVERY == 0
        H = hist.live() + [Dn]
        if refresh:
            dev.lincomb(R, [R, Dn], [1.0, tau])
            core.constraint_values(R)
            core.c_times(R, core.CR)
        out = core.grad_value(R, lam, rho, scale, g, gscr, yscr, H, D=Dn, CD=core.CD, tau=tau,
                              refresh=refresh)
        L = scale * out["crr"] + out["lres"] + 0.5 * rho * out["rr"]
        gg = out["gg"]
        if not (math.isfinite(L) and math.isfinite(gg)):
            raise DivergedError("inner iteration diverged", last_iterate=R)
        gnew, ynew = gscr, yscr
        # Gram rows of the new gradient and of y against every live buffer
        for t, v in zip(H, out["gH"]):
            hist.set_dot(gnew, t, v)
        for t, v in zip(H, out["yH"]):
            hist.set_dot(ynew, t, v)
        hist.set_dot(gnew, gnew, gg)
        hist.set_dot(ynew, ynew, out["yy"])
        hist.set_dot(gnew, ynew, out["gy"])
        ys = tau * out["yd"]
        accepted, evicted = hist.push(Dn, ynew, tau, ys)
        hist.forget(g)
        gscr = g
        g = gnew
        if accepted:
            yscr = evicted[1] if evicted else pool.get()
            if evicted:
                pool.put(evicted[0])
        else:
            hist.forget(Dn)
            hist.forget(ynew)
            pool.put(Dn)
            yscr = ynew
        iterations = it + 1
        if recorder is not None:
            recorder.record("alm", L, math.sqrt(out["rr"]) / (1.0 + b1), gnorm, rho, None)
    return finish(True)


def alm_inner(R, dual: DualVector, ops, *, scale=1.0, tol=1e-8, max_iter=500,
              reduce_factor=None, lbfgs_memory=8, recorder=None, core=None) -> InnerResult:
    """Minimise the Lagrangian over R for fixed multipliers (alm.py:268)."""
    host = not isinstance(R, torch.Tensor)
    r = R.shape[1]
    Rd, ld = _prep(ops, R)
    Rd = Rd.clone() if Rd is R else Rd
    core = core or AlmCore(ops, Rd.shape[0], ld)
    lam = _lam_dev(ops, dual.lam)
    res = _inner(core, Rd, lam, dual.rho, scale, tol, max_iter, reduce_factor, lbfgs_memory,
                 _RankRecorder(recorder, r))
    if host:
        res.R = res.R[:, :r].cpu().numpy()
        res.ax = res.ax.cpu().numpy()
    return res


class _RankRecorder:
    """Fills in the rank column of trace records."""

    def __init__(self, rec, r):
        self.rec, self.r = rec, r

    def record(self, stage, obj, err1, metric, rho, rank, t=None):
        if self.rec is not None:
            self.rec.record(stage, obj, err1, metric, rho, self.r if rank is None else rank, t=t)

    def __bool__(self):
        return self.rec is not None


@dataclass
class AlmResult:
    R: object
    outer_iterations: int
    inner_iterations: int
    err1: float
    ax: object
    hit_deadline: bool = False


def residual_norm(ops, ax, at=300):
    """||ax - b|| via one reduction."""
    dev = ops.dev
    dev.lincomb(None, [ax, ops.b], [1.0, -1.0], dots=[("out", "out")], at=at)
    return math.sqrt(float(dev.fetch(at + 1)[at]))


def alm_outer(R, dual: DualVector, ops, *, scale=1.0, switch_threshold=1e-3, outer_cap=50,
              inner_cap=500, inner_tol_floor=1e-8, lbfgs_memory=8, rho_growth=2.0, rho_max=1e8,
              escalate=None, recorder=None, deadline=None, rank=None, own=False) -> AlmResult:
    """Inner solves + dual ascent until the primal switch threshold (alm.py:337).

    ``dual.lam`` is updated in place on the device when it is a device tensor.
    ``escalate(R_dev, r) -> (R_dev_new, r_new) or None`` raises the rank.
    ``own``: the caller hands R over (the driver): it is iterated in place instead of
    copied, saving one factor of HBM.
    """
    host = not isinstance(R, torch.Tensor)
    dev = ops.dev
    p = ops.problem
    Rd, ld = _prep(ops, R)
    if Rd is R and not own:
        Rd = Rd.clone()
    r = R.shape[1] if rank is None else rank
    lam = _lam_dev(ops, dual.lam)
    if lam is not dual.lam:
        lam = lam.clone()
    core = AlmCore(ops, Rd.shape[0], ld)
    ax = core.constraint_values(Rd)
    pmeas = residual_norm(ops, ax) / (1.0 + p.b_norminf)
    inner_total = 0
    cap_streak = 0
    outer = 0
    hit_deadline = False
    res = dev.empty(p.m)
    while pmeas > switch_threshold and outer < outer_cap:
        if deadline is not None and time.perf_counter() > deadline:
            hit_deadline = True
            break
        reduce = max(1e-4, min(1e-2, 0.1 * pmeas))
        inner = _inner(core, Rd, lam, dual.rho, scale, inner_tol_floor, inner_cap, reduce,
                       lbfgs_memory, _RankRecorder(recorder, r))
        ax = inner.ax
        inner_total += inner.iterations
        dev.lincomb(res, [ax, ops.b], [1.0, -1.0], dots=[("out", "out")], at=310)
        dev.lincomb(lam, [lam, res], [1.0, dual.rho])
        new_pmeas = math.sqrt(float(dev.fetch(311)[310])) / (1.0 + p.b_norminf)
        if new_pmeas > 0.9 * pmeas:
            dual.rho = min(dual.rho * rho_growth, rho_max)
        pmeas = new_pmeas
        outer += 1
        cap_streak = cap_streak + 1 if inner.hit_cap else 0
        if cap_streak >= 2 and escalate is not None:
            grown = escalate(Rd, r)          # -> (R_new, r_new) or None
            if grown is not None:
                Rd, r = grown
                ld = Rd.shape[1]
                core = AlmCore(ops, Rd.shape[0], ld)
                ax = core.constraint_values(Rd)
            cap_streak = 0
    err1 = residual_norm(ops, ax) / (1.0 + p.b_norm1)
    if host:
        dual.lam = lam.cpu().numpy()
        return AlmResult(R=Rd[:, :r].cpu().numpy(), outer_iterations=outer,
                         inner_iterations=inner_total, err1=err1, ax=ax.cpu().numpy(),
                         hit_deadline=hit_deadline)
    dual.lam = lam
    res_obj = AlmResult(R=Rd, outer_iterations=outer, inner_iterations=inner_total, err1=err1,
                        ax=ax, hit_deadline=hit_deadline)
    res_obj.rank = r
    return res_obj

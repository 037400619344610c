"""CPU oracle for the lrsdp solve path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

This module restates, in plain numpy/scipy, the algorithm of the reference
solver at /root/reference/pkg/src/lrsdp (an un-accelerated CPU package):
the fused/column-compressed constraint operator, the Burer-Monteiro ALM
stage (L-BFGS two-loop + exact quartic line search), the splitting ADMM
stage (matrix-free CG half-steps), the Lanczos dual-infeasibility estimate,
the error metrics and the two-stage driver with re-optimisation.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this file, and only as the checker / the reference arm.
The product path (``paper_2407_15049_b200``) never imports it.

Pinning: ``tests/golden/make_golden.py`` runs the reference package itself
(imported from /root/reference in the build container) on seeded inputs and
stores its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this restatement against those fixtures (bit-for-bit on the operator
layer, per-iteration traces on full solves).

Every function names the reference file:line it follows. The numerical
operations are kept in the same order as the reference so that the oracle
reproduces it exactly on the same inputs (same numpy/scipy build).
"""

from __future__ import annotations

import math
import time
from collections import deque

import numpy as np
import scipy.sparse as sp
from scipy.linalg import eigh_tridiagonal

# problem.py:37-38
DENSE_C_THRESHOLD = 0.25
DENSE_C_MAX_N = 4096


class OracleDiverged(RuntimeError):
    def __init__(self, msg, last=None):
        super().__init__(msg)
        self.last = last


class OracleSpd(RuntimeError):
    pass


# ----------------------------------------------------------------------------
# problem helpers (duck-typed: any object with n, m, C{rows,cols,vals},
# a_con, a_row, a_col, a_val, b, maximize)
# ----------------------------------------------------------------------------

def c_nnz_full(p):
    """problem.py:65 -- nonzeros of the mirrored objective."""
    return len(p.C.vals) + int(np.count_nonzero(p.C.rows != p.C.cols))


def is_dense_c(p):
    """problem.py:211 -- small, filled objectives are stored dense."""
    return p.n <= DENSE_C_MAX_N and c_nnz_full(p) > DENSE_C_THRESHOLD * p.n * p.n


def norms(p):
    """problem.py:206-208 -- ||b||_1, ||b||_inf, ||vec C||_1."""
    b = np.asarray(p.b, dtype=np.float64)
    off = p.C.rows != p.C.cols
    cn = float(np.sum(np.abs(p.C.vals)) + np.sum(np.abs(p.C.vals[off])))
    return float(np.sum(np.abs(b))), (float(np.max(np.abs(b))) if len(b) else 0.0), cn


def nnz_a_full(p):
    """problem.py:226."""
    return len(p.a_val) + int(np.count_nonzero(p.a_row != p.a_col))


def _mirror(n, tag, r, c, v):
    """linops.py:130 -- upper-triangle triplets to full-vectorisation codes."""
    o = r != c
    return (np.concatenate([r * n + c, c[o] * n + r[o]]),
            np.concatenate([tag, tag[o]]),
            np.concatenate([v, v[o]]))


# Set operations of the reference's linops.py:139 compress, by explicit sorts: the same
# arrays as np.unique / np.union1d / np.searchsorted, which on this numpy (2.3, hash-based
# unique; random-order binary searches) take minutes at the bench's 10^7 rows.

def _unique_inverse(a):
    """np.unique(a, return_inverse=True)."""
    a = np.asarray(a)
    order = np.argsort(a, kind="stable")
    s = a[order]
    flag = np.empty(s.size, dtype=bool)
    flag[:1] = True
    np.not_equal(s[1:], s[:-1], out=flag[1:])
    inv = np.empty(a.size, dtype=np.intp)
    inv[order] = np.cumsum(flag) - 1
    return s[flag], inv


def _union_sorted(a, b):
    """np.union1d(a, b)."""
    s = np.sort(np.concatenate([np.ravel(a), np.ravel(b)]))
    if s.size == 0:
        return s
    flag = np.empty(s.size, dtype=bool)
    flag[0] = True
    np.not_equal(s[1:], s[:-1], out=flag[1:])
    return s[flag]


def _searchsorted(sorted_arr, q):
    """np.searchsorted(sorted_arr, q) with the queries visited in sorted order."""
    q = np.asarray(q)
    order = np.argsort(q, kind="stable")
    out = np.empty(q.size, dtype=np.intp)
    out[order] = np.searchsorted(sorted_arr, q[order])
    return out


def c_dense(p):
    M = np.zeros((p.n, p.n))
    M[p.C.rows, p.C.cols] = p.C.vals
    M[p.C.cols, p.C.rows] = p.C.vals
    return M


def c_csr(p):
    """linops.py:197 -- symmetric CSR of the objective."""
    o = p.C.rows != p.C.cols
    r = np.concatenate([p.C.rows, p.C.cols[o]])
    c = np.concatenate([p.C.cols, p.C.rows[o]])
    v = np.concatenate([p.C.vals, p.C.vals[o]])
    return sp.csr_matrix((v, (r, c)), shape=(p.n, p.n))


# ----------------------------------------------------------------------------
# operator layer (linops.py)
# ----------------------------------------------------------------------------

class OracleOps:
    """linops.py:139 compress + linops.py:220 build_operators, in one object.

    cols:   m x K CSR over the retained (i, j) positions, lexicographic
    imap/jmap: position of each retained column
    slot:   position of each retained column inside the support Omega
    sup_i/sup_j: Omega (union of constraint positions and C's support)
    At:     |Omega| x m CSR (transpose rows aligned to Omega)
    cvals:  C's values on Omega (zero elsewhere)
    """

    def __init__(self, p, dense_c=None):
        n, m = p.n, p.m
        self.p = p
        self.n, self.m = n, m
        if dense_c is None:
            dense_c = is_dense_c(p)
        codes, cons, vals = _mirror(n, p.a_con, p.a_row, p.a_col, p.a_val)
        uniq, colidx = _unique_inverse(codes)
        self.K = len(uniq)
        self.rows = sp.csr_matrix((vals, (cons, colidx)), shape=(m, self.K))
        self.imap, self.jmap = uniq // n, uniq % n
        if dense_c:
            sup = uniq
            self.slot = np.arange(self.K, dtype=np.int64)
            self.At = sp.csr_matrix((vals, (colidx, cons)), shape=(self.K, m))
            self.cvals = np.zeros(self.K)
            self.dense = c_dense(p)
        else:
            ccodes, _, cv = _mirror(n, np.zeros(len(p.C.vals), dtype=np.int64),
                                    p.C.rows, p.C.cols, p.C.vals)
            sup = _union_sorted(uniq, ccodes)
            self.slot = _searchsorted(sup, uniq)
            self.At = sp.csr_matrix((vals, (self.slot[colidx], cons)), shape=(len(sup), m))
            self.cvals = np.zeros(len(sup))
            self.cvals[_searchsorted(sup, ccodes)] = cv
            self.dense = None
        self.sup_i, self.sup_j = sup // n, sup % n
        self.indptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.sup_i, minlength=n), out=self.indptr[1:])
        self.c_mat = self.dense if self.dense is not None else c_csr(p)
        self.b = np.asarray(p.b, dtype=np.float64)
        self.b1, self.binf, self.cnorm1 = norms(p)

    # linops.py:49
    def sddmm(self, U, V):
        return np.einsum("kr,kr->k", U[self.imap], V[self.jmap])

    # linops.py:62
    def apply(self, x):
        return self.rows @ x

    # linops.py:70
    def A(self, U, V):
        return self.apply(self.sddmm(U, V))

    # linops.py:93
    def At_apply(self, y):
        return self.At @ y

    # linops.py:100
    def assemble(self, lam=None, extra=None, c_coeff=1.0):
        data = np.zeros(len(self.sup_i))
        if lam is not None:
            data += self.At_apply(lam)
        if extra is not None:
            data += self.At_apply(extra)
        if self.dense is not None and c_coeff != 0.0:
            S = c_coeff * self.dense
            S[self.sup_i, self.sup_j] += data
            return S
        if self.dense is None and c_coeff != 0.0:
            data += c_coeff * self.cvals
        return sp.csr_matrix((data, self.sup_j.copy(), self.indptr), shape=(self.n, self.n))

    # linops.py:215
    def objective(self, U, V):
        return float(np.sum((self.c_mat @ V) * U))


# ----------------------------------------------------------------------------
# ALM stage (alm.py)
# ----------------------------------------------------------------------------

def lbfgs_two_loop(g, pairs):
    """alm.py:98 -- two-loop recursion, identity seed; pairs oldest first."""
    D = -g.copy()
    alph = []
    for s, y, beta in reversed(pairs):
        a = beta * float(np.sum(s * D))
        D -= a * y
        alph.append(a)
    for (s, y, beta), a in zip(pairs, reversed(alph)):
        D += (a - beta * float(np.sum(y * D))) * s
    return D


def push_pair(pairs, cap, s, y):
    """alm.py:84 -- keep (s, y, 1/<y,s>) only under positive curvature."""
    ys = float(np.sum(y * s))
    if ys > 0.0:
        pairs.append((s, y, 1.0 / ys))
        return True
    return False


def quartic(ops, R, D, lam, rho, scale, ax, CR, CD):
    """alm.py:135 -- coefficients (a1..a4) and q-vectors of the exact line search."""
    q0 = ops.b - ax
    q1 = ops.apply(ops.sddmm(R, D) + ops.sddmm(D, R))
    q2 = ops.A(D, D)
    p1 = scale * float(np.sum(CD * R) + np.sum(CR * D))
    p2 = scale * float(np.sum(CD * D))
    w = -lam + rho * q0
    a1 = 0.5 * rho * float(np.dot(q2, q2))
    a2 = rho * float(np.dot(q1, q2))
    a3 = p2 - float(np.dot(w, q2)) + 0.5 * rho * float(np.dot(q1, q1))
    a4 = p1 - float(np.dot(w, q1))
    return (a1, a2, a3, a4), q1, q2


def cubic_real_roots(c3, c2, c1, c0):
    """alm.py:166 -- depressed-cubic closed form plus two Newton polishes."""
    b2, b1, b0 = c2 / c3, c1 / c3, c0 / c3
    sh = b2 / 3.0
    P = b1 - b2 * b2 / 3.0
    Q = b0 - b2 * b1 / 3.0 + 2.0 * b2 ** 3 / 27.0
    disc = -4.0 * P ** 3 - 27.0 * Q ** 2
    if abs(P) < 1e-300 and abs(Q) < 1e-300:
        ts = [0.0]
    elif disc > 0.0:
        mf = 2.0 * math.sqrt(-P / 3.0)
        arg = min(1.0, max(-1.0, 3.0 * Q / (P * mf)))
        th = math.acos(arg) / 3.0
        ts = [mf * math.cos(th - 2.0 * math.pi * k / 3.0) for k in range(3)]
    else:
        hq = -0.5 * Q
        rad = math.sqrt(max(0.0, Q * Q / 4.0 + P ** 3 / 27.0))
        u = math.copysign(abs(hq + rad) ** (1.0 / 3.0), hq + rad)
        v = math.copysign(abs(hq - rad) ** (1.0 / 3.0), hq - rad)
        ts = [u + v]
    out = []
    for t in ts:
        x = t - sh
        for _ in range(2):
            f = ((c3 * x + c2) * x + c1) * x + c0
            df = (3.0 * c3 * x + 2.0 * c2) * x + c1
            if df != 0.0 and math.isfinite(f) and math.isfinite(df):
                x -= f / df
        out.append(x)
    return out


def quartic_value(a, t):
    """alm.py:128."""
    return ((a[0] * t + a[1]) * t + a[2]) * t * t + a[3] * t


def step_length(a):
    """alm.py:202 -- minimiser of the ray quartic, (tau, zero_direction)."""
    a1, a2, a3, a4 = a
    if a1 == 0.0 and a2 == 0.0 and a3 == 0.0 and a4 == 0.0:
        return 0.0, True
    if a1 != 0.0:
        cand = cubic_real_roots(4.0 * a1, 3.0 * a2, 2.0 * a3, a4) + [0.0]
    elif a2 != 0.0:
        disc = a3 * a3 - 3.0 * a2 * a4
        cand = [0.0]
        if disc >= 0.0:
            for sg in (1.0, -1.0):
                t = (-a3 + sg * math.sqrt(disc)) / (3.0 * a2)
                if 6.0 * a2 * t + 2.0 * a3 > 0.0:
                    cand.append(t)
    elif a3 != 0.0:
        cand = [-a4 / (2.0 * a3)] if a3 > 0.0 else [0.0]
    else:
        cand = [0.0]
    vals = [quartic_value(a, t) if math.isfinite(t) else math.inf for t in cand]
    vmin = min(vals)
    tol = 1e-12 * (1.0 + abs(vmin))
    tied = sorted((t for t, v in zip(cand, vals) if v <= vmin + tol), key=lambda t: (abs(t), -t))
    return tied[0], False


def alm_grad(ops, R, lam, rho, scale, ax):
    """alm.py:239 -- 2 S R, S = scale C + A*(lam + rho (A(RR^T) - b))."""
    w = lam + rho * (ax - ops.b)
    return 2.0 * (ops.assemble(lam=w, c_coeff=scale) @ R)


def alm_val(ops, R, lam, rho, scale, ax, CR):
    """alm.py:248."""
    res = ax - ops.b
    return (scale * float(np.sum(CR * R)) + float(np.dot(lam, res))
            + 0.5 * rho * float(np.dot(res, res)))


class Tracer:
    """driver.py:144 -- (stage, counter, user objective, err1, metric, rho, rank)."""

    def __init__(self, maximize):
        self.rows = []
        self.scale = 1.0
        self.sign = -1.0 if maximize else 1.0

    def record(self, stage, obj, err1, metric, rho, rank):
        self.rows.append((stage, len(self.rows) + 1, self.sign * obj / self.scale,
                          err1, metric, rho, rank))


def alm_inner(ops, R, st, *, scale=1.0, tol=1e-8, max_iter=500, reduce_factor=None,
              memory=8, tracer=None):
    """alm.py:268 -- L-BFGS + exact line search for fixed multipliers.

    ``st`` is a dict holding 'lam' and 'rho'. Returns (R, iters, hit_cap, ax).
    """
    lam, rho = st["lam"], st["rho"]
    R = np.array(R, copy=True)
    ax = ops.A(R, R)
    CR = ops.c_mat @ R
    pairs = deque(maxlen=memory)
    g = alm_grad(ops, R, lam, rho, scale, ax)
    L = alm_val(ops, R, lam, rho, scale, ax, CR)
    if not (np.isfinite(L) and np.all(np.isfinite(g))):
        raise OracleDiverged("non-finite Lagrangian at inner start", R)
    g0 = float(np.linalg.norm(g))
    iters = 0
    for it in range(max_iter):
        gn = float(np.linalg.norm(g))
        if gn / (1.0 + abs(L)) <= tol:
            return R, iters, False, ax
        if reduce_factor is not None and gn <= reduce_factor * g0:
            return R, iters, False, ax
        D = lbfgs_two_loop(g, pairs)
        CD = ops.c_mat @ D
        a, q1, q2 = quartic(ops, R, D, lam, rho, scale, ax, CR, CD)
        tau, zero = step_length(a)
        if zero or tau == 0.0:
            return R, iters, False, ax
        R = R + tau * D
        ax = ax + tau * q1 + tau * tau * q2
        CR = CR + tau * CD
        if (it + 1) % 50 == 0:          # alm.py:29,309 refresh cadence
            ax = ops.A(R, R)
            CR = ops.c_mat @ R
        gnew = alm_grad(ops, R, lam, rho, scale, ax)
        L = alm_val(ops, R, lam, rho, scale, ax, CR)
        if not (np.isfinite(L) and np.all(np.isfinite(gnew))):
            raise OracleDiverged("inner iteration diverged", R)
        push_pair(pairs, memory, tau * D, gnew - g)
        g = gnew
        iters = it + 1
        if tracer is not None:
            tracer.record("alm", L, float(np.linalg.norm(ax - ops.b)) / (1.0 + ops.b1),
                          gn, rho, R.shape[1])
    return R, iters, True, ax


def alm_outer(ops, R, st, *, scale=1.0, switch=1e-3, outer_cap=50, inner_cap=500,
              tol_floor=1e-8, memory=8, growth=2.0, rho_max=1e8, escalate=None,
              tracer=None, deadline=None):
    """alm.py:337 -- inner solves + dual ascent until the switch threshold."""
    ax = ops.A(R, R)
    pm = float(np.linalg.norm(ax - ops.b)) / (1.0 + ops.binf)
    inner_total = streak = outer = 0
    hit_deadline = False
    while pm > switch and outer < outer_cap:
        if deadline is not None and time.perf_counter() > deadline:
            hit_deadline = True
            break
        red = max(1e-4, min(1e-2, 0.1 * pm))
        R, its, cap, ax = alm_inner(ops, R, st, scale=scale, tol=tol_floor, max_iter=inner_cap,
                                    reduce_factor=red, memory=memory, tracer=tracer)
        inner_total += its
        res = ax - ops.b
        st["lam"] = st["lam"] + st["rho"] * res
        new = float(np.linalg.norm(res)) / (1.0 + ops.binf)
        if new > 0.9 * pm:
            st["rho"] = min(st["rho"] * growth, rho_max)
        pm = new
        outer += 1
        streak = streak + 1 if cap else 0
        if streak >= 2 and escalate is not None:
            Rn = escalate(R)
            if Rn is not None:
                R = Rn
                ax = ops.A(R, R)
            streak = 0
    err1 = float(np.linalg.norm(ax - ops.b)) / (1.0 + ops.b1)
    return dict(R=R, outer=outer, inner=inner_total, err1=err1, ax=ax, hit_deadline=hit_deadline)


# ----------------------------------------------------------------------------
# ADMM stage (admm.py)
# ----------------------------------------------------------------------------

def half_apply(ops, W, Wf, rho):
    """admm.py:45 -- rho (A*(A(W Wf^T)) Wf + W)."""
    y = ops.A(W, Wf)
    return rho * ((ops.assemble(lam=y, c_coeff=0.0) @ Wf) + W)


def half_rhs(ops, Wf, lam, rho, scale=1.0, Sb=None):
    """admm.py:52."""
    if Sb is None:
        Sb = ops.assemble(lam=-lam, extra=rho * ops.b, c_coeff=-scale)
    return (Sb @ Wf) + rho * Wf


def cg(x0, op, rhs, eps, max_iter):
    """admm.py:65 -- CG on matrix iterates with Frobenius products."""
    x = np.array(x0, copy=True)
    r = rhs - op(x)
    rn = float(np.linalg.norm(r))
    if rn <= eps:
        return x, 0, rn
    p = r.copy()
    qr = float(np.sum(r * r))
    its = 0
    for k in range(max_iter):
        Q = op(p)
        pq = float(np.sum(p * Q))
        if not np.isfinite(pq):
            raise OracleDiverged("CG produced non-finite curvature", x)
        if pq <= 0.0:
            raise OracleSpd(f"non-positive curvature {pq:.3e} in CG")
        al = qr / pq
        x += al * p
        r -= al * Q
        qn = float(np.sum(r * r))
        rn = float(np.sqrt(qn))
        its = k + 1
        if rn <= eps:
            break
        p = r + (qn / qr) * p
        qr = qn
    if not np.all(np.isfinite(x)):
        raise OracleDiverged("CG iterate diverged", x)
    return x, its, rn


def admm_step(ops, S, *, scale=1.0, cg_cap=200, rel_floor=1e-10, coeff=0.05):
    """admm.py:136 -- U half-solve, V half-solve, dual ascent. S: state dict."""
    rho = S["rho"]
    if S["ax"] is None:
        S["ax"] = ops.A(S["U"], S["V"])
    pm = float(np.linalg.norm(S["ax"] - ops.b)) / (1.0 + ops.binf)
    rel = max(rel_floor, min(1e-2, coeff * pm))
    Sb = ops.assemble(lam=-S["lam"], extra=rho * ops.b, c_coeff=-scale)
    V = S["V"]
    rhs = (Sb @ V) + rho * V
    eu = max(rel * float(np.linalg.norm(rhs)), 1e-300)
    U, iu, ru = cg(S["U"], lambda W: half_apply(ops, W, V, rho), rhs, eu, cg_cap)
    S["U"], S["ax"] = U, None
    rhs = (Sb @ U) + rho * U
    ev = max(rel * float(np.linalg.norm(rhs)), 1e-300)
    V, iv, rv = cg(S["V"], lambda W: half_apply(ops, W, U, rho), rhs, ev, cg_cap)
    S["V"] = V
    S["ax"] = ops.A(S["U"], S["V"])
    S["lam"] = S["lam"] + rho * (S["ax"] - ops.b)
    cap = (iu >= cg_cap and ru > eu) or (iv >= cg_cap and rv > ev)
    return iu, iv, ru, rv, cap


def admm_run(ops, S, *, scale=1.0, eps=1e-5, gap_eps=None, min_steps=0, step_cap=20000,
             cg_cap=200, mu=10.0, tau_b=2.0, every=5, rho_min=1e-6, rho_max=1e8,
             window=60, ratio=0.995, escalate=None, tracer=None, deadline=None):
    """admm.py:184 -- ADMM steps with residual balancing and gap-stall exit."""
    b, b1, binf = ops.b, ops.b1, ops.binf

    def meas():
        if S["ax"] is None:
            S["ax"] = ops.A(S["U"], S["V"])
        pn = float(np.linalg.norm(S["ax"] - b))
        return pn, pn / (1.0 + b1), pn / (1.0 + binf)

    def gap():
        obj = ops.objective(S["U"], S["V"])
        lb = float(np.dot(-S["lam"] / scale, b))
        return abs(obj - lb) / (1.0 + abs(obj) + abs(lb))

    pn, e1, p0 = meas()
    g3 = gap() if gap_eps is not None else None
    if p0 <= eps and (gap_eps is None or g3 < gap_eps) and min_steps == 0:
        return dict(steps=0, err1=e1, p0=p0, cg=0, hit_deadline=False, hit_cap=False,
                    stalled=False, gap=g3)
    cg_total = streak = steps = 0
    hit_deadline = stalled = False
    hist = deque(maxlen=window)
    for step in range(1, step_cap + 1):
        if deadline is not None and time.perf_counter() > deadline:
            hit_deadline = True
            break
        Up, Vp = S["U"], S["V"]
        iu, iv, ru, rv, cap = admm_step(ops, S, scale=scale, cg_cap=cg_cap)
        cg_total += iu + iv
        steps = step
        pn, e1, p0 = meas()
        g3 = gap() if gap_eps is not None else None
        if tracer is not None:
            obj = scale * float(np.sum((ops.c_mat @ S["V"]) * S["U"]))
            tracer.record("admm", obj, e1, max(ru, rv), S["rho"], S["U"].shape[1])
        if p0 <= eps and (gap_eps is None or g3 < gap_eps) and step >= min_steps:
            break
        if gap_eps is not None and p0 <= eps:
            hist.append(g3)
            if len(hist) == window and hist[-1] > ratio * hist[0]:
                stalled = True
                break
        else:
            hist.clear()
        if step % every == 0:
            ds = S["rho"] * (float(np.linalg.norm(S["U"] - Up)) + float(np.linalg.norm(S["V"] - Vp)))
            if pn > mu * ds:
                S["rho"] = min(S["rho"] * tau_b, rho_max)
            elif ds > mu * pn:
                S["rho"] = max(S["rho"] / tau_b, rho_min)
        streak = streak + 1 if cap else 0
        if streak >= 2 and escalate is not None:
            pair = escalate(S["U"], S["V"])
            if pair is not None:
                S["U"], S["V"], S["ax"] = pair[0], pair[1], None
            streak = 0
    return dict(steps=steps, err1=e1, p0=p0, cg=cg_total, hit_deadline=hit_deadline,
                hit_cap=streak > 0, stalled=stalled, gap=g3)


# ----------------------------------------------------------------------------
# spectral (spectral.py)
# ----------------------------------------------------------------------------

def lanczos_min(apply_s, n, seed, max_basis=300):
    """spectral.py:28 -- Lanczos, full reorthogonalisation applied twice."""
    rng = np.random.default_rng(seed)
    kmax = min(n, max_basis)
    Q = np.zeros((kmax, n))
    al = np.zeros(kmax)
    be = np.zeros(max(kmax - 1, 0))
    q = rng.standard_normal(n)
    q /= np.linalg.norm(q)
    k = 0
    while k < kmax:
        Q[k] = q
        u = apply_s(q)
        al[k] = float(np.dot(q, u))
        r = u - al[k] * q
        if k > 0:
            r -= be[k - 1] * Q[k - 1]
        r -= Q[:k + 1].T.dot(Q[:k + 1].dot(r))
        r -= Q[:k + 1].T.dot(Q[:k + 1].dot(r))
        k += 1
        beta = float(np.linalg.norm(r))
        if k == kmax or beta <= 1e-14 * max(abs(al[:k]).max(), 1.0):
            break
        be[k - 1] = beta
        q = r / beta
    th, y = eigh_tridiagonal(al[:k], be[:k - 1], select="i", select_range=(0, 0))
    th = float(th[0])
    v = Q[:k].T.dot(y[:, 0])
    vn = np.linalg.norm(v)
    if vn > 0:
        v /= vn
    return th, float(np.linalg.norm(apply_s(v) - th * v)), k


def min_eig(apply_s, n, tol=1e-7, seed=0, max_basis=300):
    """spectral.py:67 -- one restart from seed+1 if the Ritz residual fails."""
    th, res, k = lanczos_min(apply_s, n, seed, max_basis)
    if res > tol * (1.0 + abs(th)):
        th2, res2, k2 = lanczos_min(apply_s, n, seed + 1, max_basis)
        if res2 < res:
            th, res, k = th2, res2, k2
    return th, res, res <= tol * (1.0 + abs(th)), k


def dual_infeas(ops, lam, tol=1e-7, seed=0):
    """spectral.py:82 -- |min(0, sigma_min(C - A*(lam)))| / (1 + ||vec C||_1)."""
    S = ops.assemble(lam=-np.asarray(lam), c_coeff=1.0)
    th, res, ok, k = min_eig(lambda v: S @ v, ops.n, tol=tol, seed=seed)
    return abs(min(0.0, th)) / (1.0 + ops.cnorm1), ok, th


# ----------------------------------------------------------------------------
# driver (driver.py)
# ----------------------------------------------------------------------------

def errors(ops, U, V, lam):
    """driver.py:93 -- err1, err3 and the raw primal measures (no err2)."""
    ax = ops.A(U, V)
    pn = float(np.linalg.norm(ax - ops.b))
    obj = ops.objective(U, V)
    lam = np.asarray(lam, dtype=np.float64)
    lb = float(np.dot(lam, ops.b))
    return dict(err1=pn / (1.0 + ops.b1), err3=abs(obj - lb) / (1.0 + abs(obj) + abs(lb)),
                pnorm=pn, p0=pn / (1.0 + ops.binf), obj=obj, lb=lb, err2=None,
                err2_ok=True, sigma=None)


def stop_ok(e, level, eps):
    """driver.py:113."""
    if level == 0:
        return e["p0"] <= eps
    if level == 1:
        return max(e["err1"], e["err3"]) < eps
    if e["err2"] is None:
        return False
    return max(e["err1"], e["err2"], e["err3"]) < eps


def update_rank(r, m):
    """driver.py:130."""
    return min(math.ceil(1.5 * r), math.ceil(math.sqrt(2.0 * m)))


def initial_rank(m, n, override=None):
    """driver.py:135."""
    cap = min(math.ceil(math.sqrt(2.0 * m)), n)
    if override is not None:
        return max(1, min(override, cap))
    return max(1, min(max(2, math.ceil(math.log2(2.0 * m + 1.0))), cap))


DEFAULTS = dict(eps=1e-5, reopt_level=1, max_reopts=5, reopt_factor=0.1, time_limit=10000.0,
                rank_init=None, lbfgs_memory=8, switch_threshold=None, seed=0, cg_cap=200,
                alm_inner_cap=500, alm_outer_cap=50, admm_step_cap=20000, eig_tol=1e-7)


def solve(p, **kw):
    """driver.py:222 -- ALM warm start, ADMM, re-opt rounds, final errors.

    Returns a dict with the report fields (driver.py:162) and the trace rows.
    """
    cfg = dict(DEFAULTS)
    cfg.update(kw)
    t0 = time.perf_counter()
    deadline = t0 + cfg["time_limit"]
    rng = np.random.default_rng(cfg["seed"])
    ops = OracleOps(p)
    n, m = p.n, p.m
    cap_r = min(math.ceil(math.sqrt(2.0 * m)), n)
    r0 = initial_rank(m, n, cfg["rank_init"])
    R = rng.standard_normal((n, r0)) / math.sqrt(n * r0)
    st = {"lam": np.zeros(m), "rho": max(1.0, m / math.sqrt(max(nnz_a_full(p), 1)))}
    hist_r = [r0]
    tr = Tracer(p.maximize)
    sign = -1.0 if p.maximize else 1.0
    switch = cfg["switch_threshold"] if cfg["switch_threshold"] is not None else max(100.0 * cfg["eps"], 1e-3)

    def pad(W, rn):
        return np.hstack([W, rng.standard_normal((n, rn - W.shape[1])) * (1e-3 / math.sqrt(n))])

    def esc1(W):
        rn = min(update_rank(W.shape[1], m), cap_r)
        if rn <= W.shape[1]:
            return None
        hist_r.append(rn)
        return pad(W, rn)

    def esc2(U, V):
        rn = min(update_rank(U.shape[1], m), cap_r)
        if rn <= U.shape[1]:
            return None
        hist_r.append(rn)
        return pad(U, rn), pad(V, rn)

    scale = 1.0
    rounds = 0
    status = "optimal"
    counts = dict(alm_outer=0, alm_inner=0, admm_steps=0, cg=0)
    U = V = R
    e = None
    diverged = False
    level, eps = cfg["reopt_level"], cfg["eps"]
    try:
        while True:
            tr.scale = scale
            a = alm_outer(ops, R, st, scale=scale, switch=switch, outer_cap=cfg["alm_outer_cap"],
                          inner_cap=cfg["alm_inner_cap"], memory=cfg["lbfgs_memory"],
                          escalate=esc1, tracer=tr, deadline=deadline)
            R = a["R"]
            counts["alm_outer"] += a["outer"]
            counts["alm_inner"] += a["inner"]
            st.update(U=R.copy(), V=R.copy(), ax=None)      # AdmmState shares the dual
            d = admm_run(ops, st, scale=scale, eps=eps, gap_eps=eps if level >= 1 else None,
                         min_steps=1 if rounds > 0 else 0, step_cap=cfg["admm_step_cap"],
                         cg_cap=cfg["cg_cap"], escalate=esc2, tracer=tr, deadline=deadline)
            U, V = st["U"], st["V"]
            counts["admm_steps"] += d["steps"]
            counts["cg"] += d["cg"]
            lr = -st["lam"] / scale
            e = errors(ops, U, V, lr)
            if level == 2 and e["err2"] is None and max(e["err1"], e["err3"]) < eps:
                e["err2"], e["err2_ok"], e["sigma"] = dual_infeas(ops, lr, cfg["eig_tol"], cfg["seed"])
            if a["hit_deadline"] or d["hit_deadline"] or time.perf_counter() > deadline:
                status = "timeout" if not stop_ok(e, level, eps) else "optimal"
                break
            if stop_ok(e, level, eps):
                status = "optimal"
                break
            if level == 0 or rounds >= cfg["max_reopts"]:
                status = "best_effort"
                break
            scale *= cfg["reopt_factor"]
            st["lam"] = st["lam"] * cfg["reopt_factor"]
            rounds += 1
            R = 0.5 * (U + V)
    except (OracleDiverged, OracleSpd) as exc:
        diverged = True
        status = "diverged"
        last = getattr(exc, "last", None)
        if last is not None and getattr(last, "ndim", 0) == 2:
            U = V = last
    lr = -st["lam"] / scale
    f = errors(ops, U, V, lr)
    if e is not None and e["err2"] is not None and not diverged:
        f["err2"], f["err2_ok"], f["sigma"] = e["err2"], e["err2_ok"], e["sigma"]
    else:
        f["err2"], f["err2_ok"], f["sigma"] = dual_infeas(ops, lr, cfg["eig_tol"], cfg["seed"])
    if status == "optimal" and not stop_ok(f, level, eps):
        status = "best_effort"
    return dict(status=status, objective=sign * f["obj"], err1=f["err1"], err2=f["err2"],
                err3=f["err3"], n=n, m=m, rank_final=U.shape[1], reopt_rounds=rounds,
                K=ops.K, omega_size=len(ops.sup_i), rank_history=hist_r, trace=tr.rows,
                U=U, V=V, lam=lr, time_s=time.perf_counter() - t0, **counts)

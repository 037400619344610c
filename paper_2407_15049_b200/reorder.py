"""Locality ordering of the vertices (rows) for graphs with geometric structure.

The SpMM gathers factor rows X[j] for the columns j of each row i. On a mesh
(the paper's 10^7-scale MaxCut instances are Delaunay triangulations) the
natural labelling is often scattered, so every gather is a random 208-byte
DRAM access. A reverse Cuthill-McKee order of the pattern (C and the
constraint positions) puts neighbours within ~sqrt(n) rows of each other:
the rows a tile gathers then sit in a window of well under a megabyte, which
L2 (126 MB) serves. Random graphs have no such structure and are left alone
(``locality_gain`` decides).

This is a relabelling of the SDP: X' = P X P^T. Objective, constraint values,
errors and the report are invariant; the solve runs on the permuted problem
and the factors (and, for diagonal constraints, the multipliers) are mapped
back. The reference does not reorder: trajectories agree with its own up to
summation order, like every other device path.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

from .problem import SdpProblem, SymmetricSparse


def _pattern(p):
    r = np.concatenate([p.C.rows, p.C.cols, p.a_row, p.a_col])
    c = np.concatenate([p.C.cols, p.C.rows, p.a_col, p.a_row])
    return sp.csr_matrix((np.ones(r.size, dtype=np.int8), (r, c)), shape=(p.n, p.n))


def _mean_span(r, c):
    return float(np.abs(r - c).mean()) if r.size else 0.0


def locality_order(p):
    """RCM permutation of the problem's union pattern: position k holds old row perm[k]."""
    return np.asarray(reverse_cuthill_mckee(_pattern(p), symmetric_mode=True), dtype=np.int64)


def locality_gain(p, perm):
    """Mean |i - j| of the pattern's off-diagonal entries before / after the permutation."""
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    r, c = p.C.rows, p.C.cols
    before = _mean_span(r, c)
    after = _mean_span(inv[r], inv[c])
    return before / max(after, 1.0)


def is_diag(p):
    idx = np.arange(p.m)
    return (p.m == p.n and p.a_val.size == p.m and np.array_equal(p.a_con, idx)
            and np.array_equal(p.a_row, idx) and np.array_equal(p.a_col, idx))


def permute(p, perm):
    """The SDP relabelled by ``perm`` (new row k = old row perm[k]).

    Diagonal constraints are renumbered with their rows (constraint k stays on
    row k); other constraints keep their ids. Returns (problem, inv) with
    inv[old] = new."""
    n = p.n
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n, dtype=np.int64)

    def upper(r, c):
        a, b = inv[r], inv[c]
        return np.minimum(a, b), np.maximum(a, b)

    cr, cc = upper(p.C.rows, p.C.cols)
    o = np.lexsort((cc, cr))
    C = SymmetricSparse(n, cr[o], cc[o], p.C.vals[o])
    ar, ac = upper(p.a_row, p.a_col)
    if is_diag(p):
        con = inv[p.a_con]
        b = np.asarray(p.b)[perm]
        o = np.argsort(con, kind="stable")
        q = SdpProblem(n=n, m=p.m, C=C, a_con=con[o], a_row=ar[o], a_col=ac[o], a_val=p.a_val[o], b=b,
                       maximize=p.maximize)
    else:
        q = SdpProblem(n=n, m=p.m, C=C, a_con=p.a_con.copy(), a_row=ar, a_col=ac, a_val=p.a_val.copy(),
                       b=np.asarray(p.b).copy(), maximize=p.maximize)
    return q, inv

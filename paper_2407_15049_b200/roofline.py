"""Algorithmic HBM bytes of the solve-path kernels (the roofline numerators).

Every figure counts what a kernel must move between HBM and the SMs with no
cache reuse across rows: each stored index/coefficient once, each gathered
factor row once per nonzero that references it (the graphs of the MaxCut
configs are random, so a referenced row is not in L2 when it is needed), each
written row once. Factor rows are ``ld`` fp64 values (ld = rank padded to
even, include/culorads.h). DESIGN.md section "Roofline model" states the same
formulas; bench.py divides them by CUDA-event kernel durations.
"""

from __future__ import annotations

F8 = 8      # fp64
I4 = 4      # int32 index
I8 = 8      # int64 row pointer


def constraint_eval_bytes(m, nnz_a, ld, diag=False, nprod=1, two_outputs=False):
    """cl_constraint_eval over the stacked constraint CSR (linops.py:70 apply_pair).

    Per constraint row: one row pointer + the output (+ a second output).
    Per nonzero: pi, pj, val and the two gathered factor rows of every
    product (``nprod`` = products per nonzero: 1 for A(UV^T); the line search
    evaluates X1Y1 + X2Y2 and X3Y3 on the same positions, rows R and D, i.e.
    two distinct rows per end). For diagonal constraints (MaxCut, pi == pj)
    both ends of a product are the same row of the same factor when X == Y.
    """
    per_row = I8 + F8 * (2 if two_outputs else 1)
    rows_per_nz = (1 if diag else 2) * nprod
    per_nz = 2 * I4 + F8 + rows_per_nz * ld * F8
    return m * per_row + nnz_a * per_nz


def pattern_spmm_bytes(nrows, nnz, ld, coef_bytes=F8, n_epi_in=0, write_out=True, at_entries=0):
    """cl_pattern_spmm: out = alpha S X + sum ycoef Y (linops.py:122 spmm).

    Per row: row pointer, the written row, the epilogue rows read.
    Per slot: column index, its coefficient source (cv: 8 B) and the
    gathered row of X. Adjoint coefficient rows add at_ptr per slot and
    (con, val, w[con]) per constraint entry (``at_entries``).
    """
    per_row = I8 + (ld * F8 if write_out else 0) + n_epi_in * ld * F8
    per_slot = I4 + coef_bytes + ld * F8
    return nrows * per_row + nnz * per_slot + at_entries * (I4 + 2 * F8)


def diag_update_bytes(n, ld, nh=0, refresh=True, d_distinct=True):
    """cl_diag_alm_update (MaxCut-shaped ALM step + gradient, alm.py:306-318).

    Reads ax, b, lam, a_c per row (+ q1, q2 when stepping), R, CR, D, g_old
    (+ CD when stepping) and the nh history rows; writes g, y (+ R, CR when
    stepping) and the updated constraint value. ``d_distinct`` False: the
    direction operand aliases R (the inner loop's first gradient), so it is
    not a separate HBM read.
    """
    vec = 4 + (0 if refresh else 2) + 1
    rd = 3 + (1 if d_distinct else 0) + (0 if refresh else 1) + nh
    wr = 2 + (0 if refresh else 2)
    return n * (vec * F8 + (rd + wr) * ld * F8)


def lincomb_bytes(N, nin, write_out=True):
    """cl_lincomb over N doubles with ``nin`` operands."""
    return N * F8 * (nin + (1 if write_out else 0))


def gradient_pass_bytes(ops, ld):
    """One Burer-Monteiro gradient evaluation on a diagonal-constraint problem
    (the bench step): A(RR^T), C R, then the fused w / 2 S R epilogue.

    Returns {kernel: bytes}."""
    p = ops.problem
    n, m = p.n, p.m
    nnz_a = int(ops.cop.con.val.numel())
    nnz_c = int(ops.c_mat.cpat.indices.numel())
    return {
        "constraint_eval": constraint_eval_bytes(m, nnz_a, ld, diag=ops.is_diag),
        "pattern_spmm": pattern_spmm_bytes(n, nnz_c, ld),
        "diag_alm_update": diag_update_bytes(n, ld, nh=0, refresh=True, d_distinct=False),
    }


# ---------------------------------------------------------------------------
# solver iterations (north_star: iteration rates as a fraction of the HBM roofline)
# ---------------------------------------------------------------------------

def alm_iteration_bytes(n, m, nnz_c, ld, cnt):
    """One native ALM inner iteration on a diagonal-constraint problem (alm.py:268 body,
    csrc/alm_native.cu launch sequence, no refresh) with ``cnt`` curvature pairs stored:

    * direction (alm.py:98, vector-free two-loop): one combination of g and the 2 cnt
      history rows -> D;
    * line search (alm.py:135): SpMM C D with <CD,R>, <CD,D>, <CR,D> (reads R, D, CR),
      q1/q2 over the constraint rows (R, D), the 5-operand m-vector pass;
    * step + gradient + Gram rows (alm.py:306-318): cl_diag_alm_update with nh = 2 cnt + 1.
    """
    nt = 1 + 2 * cnt
    N = n * ld
    direction = lincomb_bytes(N, nt)
    ls_spmm = pattern_spmm_bytes(n, nnz_c, ld, n_epi_in=3)
    ls_con = n * (2 * ld * F8 + F8 + 2 * F8)
    ls_vec = lincomb_bytes(m, 5)
    update = diag_update_bytes(n, ld, nh=2 * cnt + 1, refresh=False)
    return direction + ls_spmm + ls_con + ls_vec + update


def admm_step_bytes(n, m, nnz_c, ld):
    """One native ADMM step (admm.py:136, csrc/admm_native.cu in-order mode) whose two CG
    solves stop at their start: rho b - lam, the two half-step starts (SpMM C Wf with the
    rhs / initial-residual epilogue: Wf and x0 rows read, r written; the V start also stores
    C U) and the streamed step end (C U, U, V; A(UV^T), residual, dual ascent, lam.b)."""
    nlam = lincomb_bytes(m, 2)
    start = pattern_spmm_bytes(n, nnz_c, ld, n_epi_in=2) + 2 * n * F8
    end = n * (3 * ld * F8 + 6 * F8)
    return nlam + 2 * start + n * ld * F8 + end


def cg_iteration_bytes(n, ld):
    """One CG iteration of a diagonal half-step (admm.py:65 body): cl_diag_cg_apply_rows
    (r, p, Wf read, p written, the per-row coefficient written) + cl_diag_cg_step (x, p, r,
    Wf read, x, r written, the coefficient read)."""
    return n * ld * F8 * 10 + n * F8 * 3

/*
 * culorads.h -- C ABI of the B200 (sm_100a) kernels behind the lrsdp solve path.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * passed as void*. Nothing here knows about torch; the Python host
 * (paper_2407_15049_b200) allocates device memory through torch and binds
 * these symbols with ctypes. Return value: 0 on success, otherwise a
 * cudaError_t (launch failure) or a CL_E* code below (bad arguments).
 *
 * Layout conventions
 *   factor     n x r fp64 factor stored row-major with a padded leading
 *              dimension ld (ld = r rounded up to even, padding columns are
 *              zero) so one factor row is a 16-byte aligned run of ld doubles.
 *   pattern    CSR over the n x n position grid: int64 indptr[n+1], int32
 *              indices[nnz]; each slot carries its coefficient either from
 *              objective values cv[] and/or from an adjoint row (int64
 *              at_ptr[nnz+1], int32 at_con[], double at_val[]) contracted
 *              with one or two m-vectors.
 *   constraint CSR of the stacked constraint operator (m rows) with the
 *              position of every nonzero pre-resolved: int64 indptr[m+1],
 *              int32 pi[], pj[] (row/col of the n x n position), double val[].
 *
 * Reductions are deterministic: per-block partial sums in a fixed grid,
 * then one block folds the partials in a fixed order. `ws` is a device
 * scratch of CL_WS_ALLOC doubles, zero-initialised once, private to the calling
 * stream (its last word is the completion counter, left at 0 after every call).
 *
 * The one-launch (cooperative) entry points (*_fused) keep their grid-barrier
 * counter and output slot in a per-device symbol and their host-side state per
 * device (csrc/fused_state.cuh); each call holds a per-family lock for its whole
 * duration (launch + synchronize), so concurrent callers on any devices/streams
 * are serialised, never interleaved on one counter.
 */
#ifndef CULORADS_H
#define CULORADS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CL_MAXIN 20          /* operands of one streaming combination        */
#define CL_MAXDOT 48         /* dot products reduced by one launch           */
#define CL_MAXY 4            /* extra row operands of a pattern product      */
#define CL_RED_BLOCKS 1184   /* 148 SMs x 8: reduction grid upper bound       */
#define CL_WS_DOUBLES (CL_RED_BLOCKS * CL_MAXDOT)
#define CL_WS_ALLOC (CL_WS_DOUBLES + 8)   /* + completion counter */

#define CL_OK 0
#define CL_EARG 1001          /* inconsistent arguments                      */
#define CL_ENODEV 1002        /* no usable sm_100 device                     */

/* Peer-memory ghost rows of a row-sharded solve (shard.py NvlinkHaloPlan): instead of
 * a halo buffer filled by a collective, a pattern's remote column is encoded in its
 * int32 index as CL_PEER_COL(owner, row) (negative: bit 31 set) and the SpMM loads that
 * factor row in place from the owner GPU's memory over NVLink. cl_pattern.nown ==
 * CL_GHOST_PEERS marks the mode; cl_pattern.ghost then points at a HOST table of
 * CL_MAX_PEERS device addresses (rank k's row block of X as mapped in this process,
 * cl_ipc_import), which the launch copies into the kernel's parameters. The constraint
 * kernel (cl_constraint_eval_halo) takes the same mode with nown == CL_GHOST_PEERS: its
 * position indices pi/pj use the encoding and ghosts[k] is operand k's host table. */
#define CL_MAX_PEERS 8
#define CL_PEER_ROW_BITS 28
#define CL_PEER_ROW_MASK ((1u << CL_PEER_ROW_BITS) - 1u)
#define CL_GHOST_PEERS (-2)
#define CL_PEER_COL(owner, row) ((int32_t)(0x80000000u | ((uint32_t)(owner) << CL_PEER_ROW_BITS) | (uint32_t)(row)))

/* Operand index meaning "the freshly computed output" in dot specifications. */
#define CL_OUT 255

/* Streaming combination over flat arrays of N doubles (factors are flat
 * n*ld arrays; m-vectors are flat m arrays):
 *   out[k] = sum_j coef[j] * in[j][k]                  (skipped if out==NULL)
 *   dots[d] = sum_k op(da[d])[k] * op(db[d])[k]       op(CL_OUT) = out value
 * `out` may alias one of the inputs (in-place update).
 * Replaces the numpy expressions of the reference's vector algebra:
 *   lbfgs_direction two-loop (alm.py:98), R + tau*D (alm.py:306),
 *   history push <y,s> (alm.py:84), CG updates (admm.py:87-96), norms. */
#define CL_DOT_PAIRS 0      /* <= 7 inputs, <= 8 dots between arbitrary operands (da/db) */
#define CL_DOT_OUT_ALL 1    /* dots out·in[j] for every input, then out·out (nin+1 dots)  */
#define CL_DOT_FIRST_TWO 2  /* no out; [j] = in0·in[j], [CL_MAXIN+j-1] = in1·in[j] (j>=1) */

typedef struct {
    int32_t nin;
    int32_t mode;           /* CL_DOT_* */
    int32_t ndot;           /* CL_DOT_PAIRS: number of (da,db) pairs; other modes: 0 = no dots */
    const double* in[CL_MAXIN];
    double coef[CL_MAXIN];
    double* out;
    uint8_t da[CL_MAXDOT];
    uint8_t db[CL_MAXDOT];
} cl_lincomb_args;

int cl_lincomb(const cl_lincomb_args* args, int64_t N, double* dots_out, double* ws, void* stream);

/* Coefficients of an n x n pattern matrix (linops.py:100 AdjointOperator.assemble):
 *   S[s] = c_coeff * cv[s] + sum_{u in at row s} at_val[u] * w1[at_con[u]]
 *                           + sum_{u in at row s} at_val[u] * w2[at_con[u]]
 * Any of cv / at_ptr / w1 / w2 may be NULL (term dropped). */
typedef struct {
    int64_t nrows;
    const int64_t* indptr;
    const int32_t* indices;
    const double* cv;
    double c_coeff;
    const int64_t* at_ptr;
    const int32_t* at_con;
    const double* at_val;
    const double* w1;
    const double* w2;
    int64_t nnz;            /* slots (indptr[nrows]); the host knows it, the launch needs it */
    double* scratch;        /* nnz+16 doubles for assembled coefficients, or NULL */
    const double* ghost;    /* row-sharded solve: rows >= nown of X live here (halo), or NULL;
                               nown == CL_GHOST_PEERS: host table of peer row blocks (above) */
    int64_t nown;           /* rows of X owned by this rank (column j >= nown reads ghost[j-nown]) */
    const double* w1g;      /* row-sharded solve: multipliers of constraints owned by other ranks */
    const double* w2g;      /* (adjoint entry con >= mown reads w?g[con-mown]), or NULL */
    int64_t mown;
} cl_pattern;

/* Pattern times factor with a fused epilogue (linops.py:122 spmm, and the
 * products S R of alm.py:245, S V of admm.py:49/62):
 *   out[i,:] = alpha * (S X)[i,:] + sum_{j<ny} ycoef[j] * Y[j][i,:]
 *   dots[d]  = sum op(da[d]) * op(db[d])   over all n*ld entries,
 *              operand 0..ny-1 = Y[j], CL_OUT = out, 16+j = Z[j].
 * Execution: a persistent tiled kernel stages each tile's row pointers,
 * column indices and slot values in shared memory with bulk copies (TMA
 * engine, mbarrier-completed, one tile ahead), so only the factor-row
 * gathers are global loads on the critical path. Slot values are cv
 * (c_coeff folded into alpha) or, when adjoint rows are active, coefficients
 * assembled into `scratch` by a streaming pre-pass. The copies read 16-byte
 * aligned supersets: indptr, indices, cv and scratch must stay readable for
 * 16 elements past their logical end (the Python host pads every array).
 * Without scratch (adjoint rows active) the coefficients are assembled
 * inside a row-group kernel instead.                                     */
typedef struct {
    int32_t ny;
    const double* Y[CL_MAXY];
    double ycoef[CL_MAXY];
    int32_t nz;
    const double* Z[CL_MAXY];
    int32_t ndot;
    uint8_t da[8];
    uint8_t db[8];
    const double* drow;     /* optional: out[i,:] += drow[i] * dmul[i] * Y[0][i,:] (dmul NULL = 1);
                               the diagonal A*(v) term of a diagonal-constraint problem */
    const double* dmul;
} cl_epilogue;

int cl_pattern_spmm(const cl_pattern* S, const double* X, int32_t ld, double alpha,
                    const cl_epilogue* epi, double* out, double* dots_out, double* ws,
                    void* stream);

/* Fused compressed outer product + stacked constraint product
 * (linops.py:49 outer_product then linops.py:62 apply, i.e. A(X Y^T)):
 *   out1[c] = sum_{t in row c} val[t] * (X1[pi]·Y1[pj] + X2[pi]·Y2[pj])   (X2 may be NULL)
 *   out2[c] = sum_{t in row c} val[t] * (X3[pi]·Y3[pj])                   (X3 may be NULL)
 * The second output serves the line search (alm.py:153-154): q1 and q2
 * from one pass over the constraint nonzeros. */
int cl_constraint_eval(int64_t m, const int64_t* indptr, const int32_t* pi, const int32_t* pj,
                       const double* val, int32_t ld,
                       const double* X1, const double* Y1, const double* X2, const double* Y2,
                       double* out1, const double* X3, const double* Y3, double* out2,
                       void* stream);

/* Diagonal-constraint form of cl_constraint_eval (constraint c is the single
 * entry a_c e_c e_c^T, m == n; MaxCut, problem.py:387 build_maxcut): the same
 * outputs from row dot products, out1[c] = a_c (X1[c].Y1[c] + X2[c].Y2[c]),
 * out2[c] = a_c X3[c].Y3[c], with no index traffic. */
int cl_diag_constraint_eval(int64_t n, const double* aval, int32_t ld, const double* X1, const double* Y1,
                            const double* X2, const double* Y2, double* out1, const double* X3, const double* Y3,
                            double* out2, void* stream);

/* Halo packing of the row-sharded solve (rows published to the other ranks
 * before an all-gather): out[i,:] = X[idx[i],:] for i < count (16-byte vector
 * path for even ld and aligned rows, scalar otherwise). */
int cl_gather_rows(const int32_t* idx, int64_t count, int32_t ld, const double* X, double* out, void* stream);

/* Half-step operator (admm.py:45 subproblem_apply) for single-entry constraints
 * (constraint c = a_c (e_i e_j^T + e_j e_i^T), or a_c e_i e_i^T; matrix completion,
 * problem.py:410): one pass over Omega_A's rows,
 *   out_i = rho (sum_{slots (i,j) of constraint c} a_c y_c Wf_j + W_i),
 *   y_c = a_c (W_lo . Wf_hi + W_hi . Wf_lo),  (lo, hi) = (min, max)(i, j),
 * i.e. A(W Wf^T) is recomputed per slot from the two gathered rows instead of a
 * separate constraint pass + coefficient assembly; dots_out[0] = <W, out>. ld <= 64. */
int cl_single_entry_apply(int64_t nrows, const int64_t* indptr, const int32_t* indices, const double* slot_a,
                          int32_t ld, const double* W, const double* Wf, double rho, double* out, double* dots_out,
                          double* ws, void* stream);
/* The same operator with W and Wf interleaved in one pair buffer P (n x 2ld, row i =
 * [W_i | Wf_i]): each slot gathers one contiguous 2ld run instead of two ld runs, which
 * touches fewer 128-byte DRAM lines (random 208-byte rows cost 2.4 lines each, a 416-byte
 * pair 3.9; tools/micro/gather_probe.cu). Same arithmetic, same thread mapping:
 * bit-identical to cl_single_entry_apply. */
int cl_single_entry_apply_pair(int64_t nrows, const int64_t* indptr, const int32_t* indices, const double* slot_a,
                               int32_t ld, const double* P, double rho, double* out, double* dots_out, double* ws,
                               void* stream);
/* P[i, half*ld : (half+1)*ld] = X[i, :] for a pair buffer P (n x 2ld). */
int cl_pair_pack(int64_t n, int32_t ld, const double* X, double* P, int32_t half, void* stream);
/* CG direction update of the pair path: p = r + beta p (cl_lincomb's arithmetic), written
 * to p (n x ld) and to P's first half. */
int cl_cg_direction_pair(int64_t n, int32_t ld, double beta, const double* r, double* p, double* P, void* stream);

/* Fused SpMM passes of the ADMM step for diagonal constraints:
 *   cl_diag_admm_cg_init: rhs = -scale C Wf + rho Wf + diag(a nlam) Wf (admm.py:52,
 *     nlam = rho b - lam) and the initial CG residual r = rhs - Q(x0) with
 *     Q(x0) = rho (a y Wf + x0), y = a <x0, Wf>  (admm.py:45/72) -- rhs and Q are
 *     never stored; dots_out[0] = ||rhs||^2, dots_out[1] = ||r||^2.
 *     cwf != NULL also stores C Wf itself (n x ld).
 *   cl_diag_admm_step_end: <C V, U> (admm.py:215), ax = A(U V^T), the residual
 *     ax - b and the dual ascent lam_new = lam + rho (ax - b) (admm.py:165-166);
 *     dots_out[0] = <C V, U>, [1] = ||ax - b||^2, [2] = lam_new . b.
 *   cl_diag_admm_step_end_rows: the same step end as one streaming pass, with the
 *     objective taken as <C U, V> from the C U the V half-step's start stored
 *     (cl_diag_admm_cg_init with Wf = U, cwf = CU): no second SpMM, no halo.
 * C carries cv values (and ghost rows in a row-sharded solve). */
int cl_diag_admm_cg_init(const cl_pattern* C, const double* Wf, const double* x0, int32_t ld, double scale, double rho,
                         const double* nlam, const double* aval, double* r, double* cwf, double* dots_out, double* ws,
                         void* stream);
int cl_diag_admm_step_end_rows(int64_t n, int32_t ld, const double* CU, const double* U, const double* V,
                               const double* aval, const double* b, const double* lam, double rho, double* ax,
                               double* lam_new, double* dots_out, double* ws, void* stream);
int cl_diag_admm_step_end(const cl_pattern* C, const double* U, const double* V, int32_t ld, const double* aval,
                          const double* b, const double* lam, double rho, double* ax, double* lam_new, double* dots_out,
                          double* ws, void* stream);

/* ADMM half-step CG for diagonal constraints (admm.py:65 cg_solve with the
 * operator of admm.py:45 subproblem_apply, A = diag(a)): one launch per
 * operator application and one per update, each factor operand read once.
 *   cl_diag_cg_apply: [p <- r + beta p if r != NULL]  y_c = a_c <p_c, Wf_c>,
 *                     Q_c = rho (a_c y_c Wf_c + p_c),  dots_out[0] = <p, Q>
 *   cl_cg_step:       x_out = x_in + alpha p,  r -= alpha Q,  dots_out[0] = <r, r>
 * (N = n*ld doubles; x_out may alias x_in). */
int cl_diag_cg_apply(int64_t n, int32_t ld, const double* aval, double rho, double beta, const double* r, double* p,
                     const double* Wf, double* Q, double* dots_out, double* ws, void* stream);
int cl_cg_step(int64_t N, double alpha, const double* x_in, double* x_out, const double* p, double* r,
               const double* Q, double* dots_out, double* ws, void* stream);
/* cl_cg_step with alpha = qr / *pq computed on the device (pq: the device reduction of
 * the preceding operator application); a non-finite or non-positive pq leaves x and r
 * untouched (cg_solve raises there, admm.py:83-86). */
int cl_cg_step_dev(int64_t N, double qr, const double* pq, const double* x_in, double* x_out, const double* p,
                   double* r, const double* Q, double* dots_out, double* ws, void* stream);

/* The same CG iteration with Q never stored: cl_diag_cg_apply_rows writes the
 * per-row coefficient coef_c = rho a_c y_c (n doubles) instead of Q, and
 * cl_diag_cg_step rebuilds Q_c = coef_c Wf_c + rho p_c with the same expression
 * while it updates x and r, so the results are bit-identical to the stored-Q
 * pair and the pass streams one n x ld operand less. alpha is taken as given,
 * or as qr / *pq on the device when pq != NULL (semantics of cl_cg_step_dev). */
int cl_diag_cg_apply_rows(int64_t n, int32_t ld, const double* aval, double rho, double beta, const double* r,
                          double* p, const double* Wf, double* coef, double* dots_out, double* ws, void* stream);
int cl_diag_cg_step(int64_t n, int32_t ld, double rho, const double* coef, const double* Wf, double alpha,
                    double qr, const double* pq, const double* x_in, double* x_out, const double* p, double* r,
                    double* dots_out, double* ws, void* stream);

/* cl_constraint_eval for a row block of a row-sharded solve: factor row
 * index >= nown of operand k (X1, Y1, X2, Y2, X3, Y3) reads ghosts[k][row-nown]
 * (the halo rows gathered from the other ranks). */
/* The line search's products (alm.py:153-154) with R and D interleaved in one pair buffer
 * P (n x 2ld, row i = [R_i | D_i]): out1 = A(R D^T + D R^T), out2 = A(D D^T) -- the
 * cl_constraint_eval call with X1=R, Y1=D, X2=D, Y2=R, X3=Y3=D, bit for bit, with each
 * position's rows gathered as one 2ld run (fewer 128-byte DRAM lines). */
int cl_constraint_eval_pair(int64_t m, const int64_t* indptr, const int32_t* pi, const int32_t* pj,
                            const double* val, int32_t ld, const double* P, double* out1, double* out2,
                            void* stream);

int cl_constraint_eval_halo(int64_t m, const int64_t* indptr, const int32_t* pi, const int32_t* pj,
                            const double* val, int32_t ld, const double* X1, const double* Y1, const double* X2,
                            const double* Y2, double* out1, const double* X3, const double* Y3, double* out2,
                            const double* const* ghosts, int64_t nown, void* stream);

/* Gathered outer product at K positions (linops.py:49), x[k] = X[imap[k]]·Y[jmap[k]]. */
int cl_sddmm(int64_t K, const int32_t* imap, const int32_t* jmap, int32_t ld,
             const double* X, const double* Y, double* x, void* stream);

/* Diagonal-constraint fast path for problems whose constraint c is the single
 * diagonal entry a_c * e_c e_c^T (m == n; MaxCut, problem.py:387): the ALM
 * step update and gradient (alm.py:306-318) become row-local and fuse into one pass.
 *   R  += tau*D;  CR += tau*CD;  ax_out[c] = ax[c] + tau*q1[c] + tau^2*q2[c]
 *   w[c] = lam[c] + rho*(ax[c]-b[c]);  g_new = 2*(w[row]*a*R + scale*CR)
 *   y = g_new - g_old        (g_old NULL: 0, y = g_new -- the inner solve's first gradient)
 * plus dots: <CR,R>, <g_new,g_new>, <y, tau D>, lam·res, res·res and the
 * multi-dots of g_new and y against up to `nh` history vectors H[]:
 *   dots[0]=<CR,R> [1]=<g,g> [2]=<y,D> [3]=lam·res [4]=res·res [5]=<y,y>
 *   [6]=<g,y>  [7+h]=<g,H_h>  [7+CL_MAXIN+h]=<y,H_h>   (dots_out: 7+2*CL_MAXIN) */
typedef struct {
    int64_t n;
    int32_t ld;
    const double* aval;          /* a_c */
    double tau, rho, scale;
    double* R; const double* D; double* CR; const double* CD;
    const double* ax; double* ax_out; const double* q1; const double* q2;
    const double* lam; const double* b;
    const double* g_old; double* g_new; double* y;
    int32_t nh;
    const double* H[CL_MAXIN];
    int32_t refresh;             /* 1: ax/CR were recomputed, skip tau updates */
} cl_diag_update_args;

int cl_diag_alm_update(const cl_diag_update_args* a, double* dots_out, double* ws, void* stream);

/* Dense block Gram helpers for the Lanczos basis (spectral.py:55-56):
 *   h[t] = sum_k Q[t][k] * v[k]            t < k_cnt   (Q row-major, ldq)
 *   v[k] -= sum_t h[t] * Q[t][k]                                          */
int cl_basis_project(const double* Q, int64_t ldq, int32_t k_cnt, int64_t n, const double* v,
                     double* h, double* ws, void* stream);
int cl_basis_subtract(const double* Q, int64_t ldq, int32_t k_cnt, int64_t n, const double* h,
                      double* v, void* stream);

/* Row-sharded solve (shard.py): the native loops below run on one rank's row
 * block when `dist` is set. The caller (the Python host, over torch.distributed)
 * supplies two hooks:
 *   exchange  halo of a factor before a C product: packs this rank's published
 *             rows of X (n_own x ld) and all-gathers them; returns the device
 *             address of the ghost rows (pattern column j >= nown reads
 *             ghost[j - nown]), NULL on failure;
 *   reduce    combines slab[0:count) over the ranks (rank-ordered sum, identical
 *             bits on every rank) into host[0:count) (pinned) after the stream's
 *             queued work; 0 on success.
 * Every reduction of the diagonal-constraint loops is a sum over rows, so with
 * the hooks the loops take the same decisions as the single-GPU ones. CG steps
 * then read <p, Q> before the update (alpha on the host), as the Python-driven
 * sharded path does. NULL `dist`: single GPU. */
typedef struct {
    void* ctx;
    const double* (*exchange)(void* ctx, const double* X, int32_t ld);
    int32_t (*reduce)(void* ctx, double* slab, double* host, int32_t count, void* stream);
    int64_t nown;
    /* Peer-memory mode (nown == CL_GHOST_PEERS): exchange returns the host table of the
     * peers' row blocks of X after a stream-ordered fence (every rank's X complete), and
     * release, called right after the product is queued, fences again so that no rank
     * overwrites its rows while a peer may still read them. NULL in the halo modes. */
    int32_t (*release)(void* ctx, void* stream);
} cl_dist_hooks;

/* One ADMM step (admm.py:136 admm_step: U half-solve, V half-solve, dual
 * ascent) for diagonal constraints, with every scalar decision of the
 * reference (tolerance schedule, cg_solve's stop/curvature/finiteness
 * tests, admm.py:65) taken in native host code between launches of the
 * kernels above. Same launches in the same order as the Python host path,
 * hence bit-identical iterates. The V half-step's start and the step end are
 * launched speculatively (assuming the CGs stop at their start, the common case)
 * so such a step costs ONE synchronize; a CG that iterates triggers the
 * recomputation of the speculative work. */
typedef struct {
    int64_t n;                 /* rows = constraints */
    int32_t ld;
    const double* aval;        /* a_c */
    const double* b;
    const double* lam;         /* multiplier at the step start */
    double* lam_new;           /* lam + rho (A(U_new V_new^T) - b) (dual ascent, out of place) */
    double* ax;                /* A(U V^T): input when ax_valid, output A(U_new V_new^T) */
    int32_t ax_valid;
    double pnorm2_known;       /* ||A(UV^T)-b||^2 of the input state, or < 0 to recompute */
    const double* U;
    const double* V;
    double* U_new;
    double* V_new;
    double* r;                 /* CG residual of the U half-step, n x ld */
    double* r_v;               /* CG residual of the V half-step (started speculatively) */
    double* p;                 /* CG direction / operator output, n x ld */
    double* Q;                 /* n x ld; its first n doubles hold the CG's per-row coefficients */
    double* cu;                /* C U_new, n x ld: written by the V half-step's start, read by the step end */
    double* nlam;              /* m-vector scratch */
    double* res;               /* m-vector scratch */
    cl_pattern cpat;           /* C (cv values) */
    double rho, scale, binf, rel_floor, primal_coeff;
    int32_t cg_cap;
    double* slab;              /* 16 device doubles for the step's reductions */
    double* host;              /* 20 pinned host doubles */
    double* ws;                /* reduction workspace (CL_WS_ALLOC doubles) */
    void* stream;
    int32_t want_balance;      /* one-launch step: also return ||U_new-U||^2, ||V_new-V||^2 */
    const cl_dist_hooks* dist; /* row-sharded solve (cl_admm_step_diag only), or NULL */
} cl_admm_diag_args;

typedef struct {
    int32_t it_u, it_v;
    double res_u, res_v, eps_u, eps_v;
    double pnorm2;             /* ||A(U_new V_new^T) - b||^2 */
    int32_t hit_cap;
    int32_t status;            /* 0 ok; 1 non-finite curvature; 2 non-positive curvature; 3 non-finite iterate */
    int32_t bad_half;          /* 0: U half-solve, 1: V half-solve */
    int32_t bad_is_new;        /* last iterate is U_new/V_new (1) or the input U/V (0) */
    double pq_bad;
    int32_t u_reused;          /* CG stopped at its start: the new U is the input U (U_new untouched) */
    int32_t v_reused;
    double objective;          /* <C, U V^T> of the new factors (admm.py:215) */
    double lam_b;              /* lam_new . b */
    int32_t err_line;          /* diagnostics: admm_native.cu line of the first failing launch */
    double du2, dv2;           /* ||U_new-U||^2, ||V_new-V||^2 when asked (want_balance), else -1 */
} cl_admm_step_stats;

int cl_admm_step_diag(const cl_admm_diag_args* a, cl_admm_step_stats* out);

/* One ADMM step (admm.py:136) for general constraints (matrix completion, SDPA
 * instances), single GPU: the launches of the Python host path (admm.admm_step's
 * generic branch with HalfStep.rhs / .cg / .apply: the right-hand side over Omega with
 * assembled coefficients, CG with the single-entry operator -- on the pair buffer when
 * `pair` is set -- or constraint pass + Omega_A product, the dual ascent in place), with
 * its scalar decisions in native code: bit-identical iterates. Writes U_new, V_new (always:
 * a CG that stops at its start copies the start), ax_new = A(U_new V_new^T) and lam (in
 * place). Stats as cl_admm_step_diag (status 1: non-finite curvature, 2: non-positive
 * curvature, 3: non-finite iterate; bad_half 0/1 = U/V). */
typedef struct {
    int64_t n, m;
    int32_t ld;
    const double* b;
    double* lam;               /* updated in place: lam + rho (A(U_new V_new^T) - b) */
    const double* ax;          /* A(U V^T) of the step start, or NULL (recomputed into ax_new) */
    double* ax_new;
    const double* U;
    const double* V;
    double* U_new;
    double* V_new;
    double* rhs;               /* n x ld */
    double* r;                 /* CG vectors, n x ld */
    double* p;
    double* Q;
    double* y;                 /* m-vector scratch (residual; the operator's constraint values) */
    double* nlam;              /* m-vector scratch */
    double* rhob;              /* m-vector scratch */
    double* pair;              /* n x 2ld pair buffer [p | Wf] (single-entry operator), or NULL */
    const int64_t* con_indptr; /* constraint CSR with resolved positions */
    const int32_t* con_pi;
    const int32_t* con_pj;
    const double* con_val;
    cl_pattern omega;          /* Omega (cv + adjoint rows, scratch) */
    cl_pattern apat;           /* Omega_A (adjoint rows, scratch) */
    const double* single_a;    /* Omega_A slot coefficients of single-entry constraints, or NULL */
    double rho, scale, binf, rel_floor, primal_coeff;
    int32_t cg_cap;
    double* slab;              /* 8 device doubles */
    double* host;              /* 8 pinned host doubles */
    double* ws;
    void* stream;
} cl_admm_generic_args;

int cl_admm_step_generic(const cl_admm_generic_args* a, cl_admm_step_stats* out);

/* ALM inner solve (alm.py:268 alm_inner) for diagonal constraints: the
 * iteration of the Python host path (vector-free L-BFGS over a host Gram
 * matrix, exact quartic line search, fused step/gradient/Gram-row update)
 * with its scalar algebra in native code; same launches and operands, hence
 * bit-identical iterates. The caller provides nbuf >= 2*memory+4 factor
 * buffers (the L-BFGS pool). Per-iteration trace records (L, err1, gnorm,
 * CLOCK_MONOTONIC seconds) go to rec[4*k..], gradient norms to gnorms[]. */
#define CL_ALM_MAXMEM 8
#define CL_ALM_MAXBUF (2 * CL_ALM_MAXMEM + 4)
#define CL_ALM_REFRESH 50      /* alm.py:29 _REFRESH_EVERY */
typedef struct {
    int64_t n;
    int32_t ld;
    int32_t memory;            /* L-BFGS pairs kept (<= CL_ALM_MAXMEM) */
    int32_t max_iter;
    double tol;
    double reduce_factor;      /* < 0: none */
    double rho, scale, b1;     /* b1 = ||b||_1 (trace err1) */
    const double* aval;
    const double* b;
    const double* lam;
    double* R;                 /* updated in place */
    double* CR;
    double* CD;
    double* ax;                /* AlmCore.ax (current constraint values on return: see ax_is_ax2) */
    double* ax2;
    double* q1;
    double* q2;
    double* wv;
    const double* zero_g;      /* g_old of the first gradient: NULL (= 0, no buffer) or a zero factor */
    int32_t nbuf;
    double* bufs[CL_ALM_MAXBUF];
    cl_pattern cpat;
    double* slab;              /* >= 64 + 7 + 2*CL_MAXIN device doubles */
    double* host;              /* same count, pinned */
    double* ws;
    void* stream;
    int32_t rec_cap;
    double* rec;               /* 4 * rec_cap host doubles */
    double* gnorms;            /* rec_cap host doubles */
    const cl_dist_hooks* dist; /* row-sharded solve (cl_alm_inner_diag only), or NULL */
    /* cl_alm_inner_generic only (general constraints: A(R R^T) by the constraint CSR, the
     * gradient's A*(w) R over Omega_A with assembled coefficients) */
    int64_t m;                 /* constraints */
    const int64_t* con_indptr; /* constraint CSR with resolved positions (cl_constraint_eval) */
    const int32_t* con_pi;
    const int32_t* con_pj;
    const double* con_val;
    cl_pattern apat;           /* Omega_A: adjoint rows (w1 = wv set here), scratch */
    double* res;               /* m doubles */
    double* pair;              /* n x 2ld pair buffer [R | D] for the line search, or NULL */
} cl_alm_inner_args;

typedef struct {
    int32_t iterations;
    int32_t n_records;
    int32_t n_gnorms;
    int32_t hit_cap;
    int32_t status;            /* 0 ok; 1 non-finite Lagrangian at start; 2 diverged inside */
    int32_t ax_is_ax2;
    int32_t err_line;
} cl_alm_inner_stats;

int cl_alm_inner_diag(const cl_alm_inner_args* a, cl_alm_inner_stats* out);
/* The same inner solve for general constraints (matrix completion, SDPA instances): the
 * launches of the Python host path's generic chain (alm.py _inner with AlmCore.grad_value's
 * generic branch and line_search), with its scalar algebra in native code: bit-identical
 * iterates. `aval` unused; m, con_*, apat, res set; `pair` optional (single-entry
 * constraints: cl_constraint_eval_pair). Single GPU (dist must be NULL). */
int cl_alm_inner_generic(const cl_alm_inner_args* a, cl_alm_inner_stats* out);
/* The same inner solve as ONE cooperative launch (csrc/alm_fused.cu) for small
 * problems: thread 0 of every block replays the scalar algebra from grid-reduced
 * values, vector passes run between grid barriers; one synchronize per inner solve.
 * Iterates agree with cl_alm_inner_diag to rounding. Requires n >= 1. */
int cl_alm_inner_diag_fused(const cl_alm_inner_args* a, cl_alm_inner_stats* out);

/* Slot values of a pattern (c_coeff cv + adjoint rows against w1/w2, linops.py:100
 * assemble) written to vals[nnz] -- the pre-pass cl_pattern_spmm runs internally. */
int cl_pattern_assemble(const cl_pattern* S, double* vals, void* stream);

/* Lanczos loop of spectral.py:28 with native control flow. S is a pattern with
 * assembled slot values (cv, no adjoint rows) applied to vectors (ld = 1); Q holds
 * k_max basis rows of ldq doubles, Q[0] the start vector. Fills alphas[0..k) and
 * betas[0..k-1) (host arrays) and returns k (the basis size) in *k_out. */
typedef struct {
    int64_t n;
    int32_t k_max;
    double breakdown;
    double* Q;
    int64_t ldq;
    double* u;
    double* r;
    double* h;                 /* k_max device doubles (Gram projections) */
    cl_pattern S;
    double* slab;              /* 2 * CL_LANCZOS_BATCH device doubles */
    double* host;              /* 2 * CL_LANCZOS_BATCH pinned host doubles */
    double* ws;
    void* stream;
    double* alphas;
    double* betas;
    double* dbeta;             /* k_max device doubles: the betas as the device sees them */
    double* dalpha;            /* k_max device doubles (cl_lanczos_loop_fused) */
} cl_lanczos_args;

/* The loop enqueues CL_LANCZOS_BATCH steps with the scalars kept on the device
 * (cl_lanczos_update), then reads their alphas and ||r||^2 at one synchronize and
 * replays the reference's stop tests in order. Steps past the stop are discarded
 * (they only touch basis rows >= k). */
#define CL_LANCZOS_BATCH 16
int cl_lanczos_loop(const cl_lanczos_args* a, int32_t* k_out);
/* The same loop as ONE cooperative launch (small n, k_max <= 4096): the stop test runs
 * on the device; one synchronize for the whole basis. Coefficients agree with
 * cl_lanczos_loop to rounding (global sums in another fixed order). */
int cl_lanczos_loop_fused(const cl_lanczos_args* a, int32_t* k_out);

/* cl_admm_step_diag as ONE cooperative launch (csrc/admm_fused.cu) for small
 * problems, where launch and round-trip latency bound the step: every phase runs
 * in one kernel between grid-wide barriers and the scalar decisions are taken on
 * the device; one synchronize per step. Same args and stats (host: 20 pinned
 * doubles); iterates equal cl_admm_step_diag's to rounding (global sums are added
 * in another fixed order). Requires n >= 1 and a C pattern with cv values only. */
int cl_admm_step_diag_fused(const cl_admm_diag_args* a, cl_admm_step_stats* out);

/* Lanczos vector updates with device-resident scalars (spectral.py:45-61):
 *   mode 0: r = u - (*alpha) qk [- (*beta) qkm1 when beta != NULL]
 *   mode 1: qn = r / sqrt(*rr), *beta_out = sqrt(*rr)
 * Bit-identical to cl_lincomb with the same coefficients taken on the host. */
int cl_lanczos_update(int32_t mode, int64_t n, const double* alpha, const double* beta, const double* u,
                      const double* qk, const double* qkm1, double* r, const double* rr, double* beta_out, double* qn,
                      void* stream);

/* L2 fetch granularity hint of the current device (cudaLimitMaxL2FetchGranularity, 0..128 bytes). */
int cl_set_l2_fetch_granularity(int32_t bytes);
int cl_get_l2_fetch_granularity(void);

/* CUDA IPC of a factor's device allocation, for the peer-memory ghost mode (replaces
 * the all-gather / all-to-all halo of shard.py HaloPlan / PeerHaloPlan: reference
 * north_star "remote factor rows come in by NCCL all-gather or halo exchange over
 * NVLink"). cl_ipc_export: the 64-byte IPC handle of the allocation holding `ptr` and
 * ptr's byte offset in it. cl_ipc_import: map a peer's handle (another process) and
 * return the allocation's base here; cl_ipc_close unmaps it. */
#define CL_IPC_HANDLE_BYTES 64
int cl_ipc_export(const void* ptr, void* handle, int64_t* offset);
int cl_ipc_import(const void* handle, void** base);
int cl_ipc_close(void* base);

/* Library identity, for load checks. */
const char* cl_version(void);
int cl_device_ok(void);

#ifdef __cplusplus
}
#endif

#endif /* CULORADS_H */

// admm_native.cu -- one ADMM step (admm.py:136 admm_step) for diagonal
// constraints, driven from native host code.
//
// At small n the host round trip after each reduction, not the GPU, bounds the
// step rate. This file takes the step's scalar decisions in C++ -- the
// tolerance schedule, cg_solve's stop / curvature / finiteness tests
// (admm.py:65), the dual ascent -- between launches of the fused kernels:
//
//   cl_diag_admm_cg_init   rhs + initial CG residual of a half-step
//   cl_diag_cg_apply_rows  CG operator (+ deferred direction update)
//   cl_diag_cg_step        x/r update
//   cl_diag_admm_step_end_rows  objective, A(UV^T), residual, dual ascent, lam.b
//                          (streams the C U the V start stored: no second SpMM)
//
// Speculation: most steps' CG solves stop at their start (the iterate is
// kept). The V half-step's start and the step end are therefore launched
// right after the U half-step's start, assuming U (then V) is kept, and the
// decisions of all three are read at ONE synchronize. When a CG does iterate
// the speculative work is recomputed with the new factor. Speculation trades
// whole passes for synchronizes, so it is used only while a pass is cheaper
// than a host round trip (n*ld <= SPEC_MAX_ELEMS); larger steps run in order. Every kernel that
// counts sees exactly the operands of the sequential order, so the iterates
// are bit-identical to the Python-driven twin (admm._admm_step_diag_py,
// tests/test_gpu_admm_native.py).

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "culorads.h"

namespace {

constexpr int64_t SPEC_MAX_ELEMS = int64_t(1) << 20;   // 8 MB per factor: a pass costs about a round trip

struct Ctx {
    const cl_admm_diag_args* a;
    cudaStream_t st;
    int rc;
    int64_t N;   // n * ld
    int line;    // source line of the first failing call (diagnostics)
};

#define CL_TRY(c, expr)                      \
    do {                                     \
        if (!(c).rc) {                       \
            (c).rc = (expr);                 \
            if ((c).rc) (c).line = __LINE__; \
        }                                    \
    } while (0)

// Reduction slots inside the caller's slab; values read at one decision point are contiguous.
enum {
    S_PM = 0,              // ||A(UV^T) - b||^2 at the step start (when not known)
    S_RHSU = 1, S_R0U = 2, // U half: ||rhs||^2, ||r0||^2
    S_XXU = 3,             // <U_new, U_new> (finiteness of the U iterate)
    S_PQ = 4, S_QN = 5,    // CG: <p, Q>, <r, r>
    S_XXV = 7,             // <V_new, V_new>
    S_E0 = 10,             // step end: objective, ||ax - b||^2, lam_new . b (3 slots)
    S_RHSV = 13, S_R0V = 14,
    S_END = 15
};

bool fetch(Ctx& c, int lo, int cnt) {
    if (c.rc) return false;
    if (c.a->dist != nullptr) {     // row-sharded: the partial sums are combined over the ranks
        if (c.a->dist->reduce(c.a->dist->ctx, c.a->slab + lo, c.a->host + lo, cnt, (void*)c.st) != 0) {
            c.rc = CL_EARG;
            c.line = __LINE__;
            return false;
        }
        return true;
    }
    cudaError_t e = cudaMemcpyAsync(c.a->host + lo, c.a->slab + lo, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                                    c.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.st);
    if (e != cudaSuccess) {
        c.rc = (int)e;
        c.line = __LINE__;
        return false;
    }
    return true;
}

double H(const Ctx& c, int slot) { return c.a->host[slot]; }

void lincomb(Ctx& c, double* out, int nin, const double* const* in, const double* coef, int64_t N, int dot_slot,
             bool dot_out_out) {
    cl_lincomb_args L;
    memset(&L, 0, sizeof(L));
    L.nin = nin;
    L.mode = CL_DOT_PAIRS;
    for (int j = 0; j < nin; ++j) {
        L.in[j] = in[j];
        L.coef[j] = coef[j];
    }
    L.out = out;
    if (dot_slot >= 0) {
        L.ndot = 1;
        L.da[0] = dot_out_out ? CL_OUT : 0;
        L.db[0] = dot_out_out ? CL_OUT : 0;
    }
    CL_TRY(c, cl_lincomb(&L, N, dot_slot >= 0 ? c.a->slab + dot_slot : nullptr, c.a->ws, (void*)c.st));
}

void copy(Ctx& c, double* dst, const double* src) {
    const double* in[1] = {src};
    const double cf[1] = {1.0};
    lincomb(c, dst, 1, in, cf, c.N, -1, false);
}

// <x, x> into slab[slot] (admm.py:98 finiteness test of the CG iterate)
void selfdot(Ctx& c, const double* x, int slot) {
    cl_lincomb_args L;
    memset(&L, 0, sizeof(L));
    L.nin = 1;
    L.mode = CL_DOT_PAIRS;
    L.in[0] = x;
    L.coef[0] = 0.0;
    L.ndot = 1;
    CL_TRY(c, cl_lincomb(&L, c.N, c.a->slab + slot, c.a->ws, (void*)c.st));
}

// half-step start: rhs (never stored), Q(x0), r = rhs - Q(x0), ||rhs||^2 and ||r||^2
// (the V half-step's start, cw = a->cu, also stores C U for the step end)
void cg_init(Ctx& c, const double* x0, const double* Wf, double* r, int slot, double* cw) {
    const cl_admm_diag_args* a = c.a;
    cl_pattern P = a->cpat;
    P.c_coeff = 1.0;
    if (a->dist != nullptr && !c.rc) {      // row-sharded: C Wf reads Wf's halo
        P.ghost = a->dist->exchange(a->dist->ctx, Wf, a->ld);
        P.nown = a->dist->nown;
        if (P.ghost == nullptr) {
            c.rc = CL_EARG;
            c.line = __LINE__;
            return;
        }
    }
    CL_TRY(c, cl_diag_admm_cg_init(&P, Wf, x0, a->ld, a->scale, a->rho, a->nlam, a->aval, r, cw, a->slab + slot,
                                   a->ws, (void*)c.st));
    // peer-memory ghosts: fence after the product that read the peers' rows of Wf
    if (a->dist != nullptr && a->dist->release != nullptr && !c.rc &&
        a->dist->release(a->dist->ctx, (void*)c.st) != 0) {
        c.rc = CL_EARG;
        c.line = __LINE__;
    }
}

// step end from the C U stored by the last V start (whose Wf is the U passed here)
void step_end(Ctx& c, const double* U, const double* V) {
    const cl_admm_diag_args* a = c.a;
    CL_TRY(c, cl_diag_admm_step_end_rows(a->n, a->ld, a->cu, U, V, a->aval, a->b, a->lam, a->rho, a->ax, a->lam_new,
                                         a->slab + S_E0, a->ws, (void*)c.st));
}

// max(v, 1e-300) with Python semantics (v is kept unless 1e-300 > v; NaN stays NaN)
double pymax_tiny(double v) { return (1e-300 > v) ? 1e-300 : v; }

// CG iterations of admm.py:65 on the diagonal operator after a start whose residual
// misses the tolerance (HalfStep._cg_diag's loop); x0 read only, result in x.
// Returns 0 ok, 1 non-finite curvature, 2 non-positive curvature.
int cg_loop(Ctx& c, const double* x0, double* x, const double* Wf, double* r, double eps, double qr, int* its_out,
            double* rnorm_out, int* last_is_x, double* pq_bad) {
    const cl_admm_diag_args* a = c.a;
    int its = 0;
    double beta = 0.0, rnorm = sqrt(qr);
    const double* xs = x0;
    *last_is_x = 0;
    for (int k = 0; k < a->cg_cap; ++k) {
        // operator application, then the update with alpha = qr / pq taken on the device:
        // pq and the new <r, r> are read together (one synchronize per iteration)
        // (Q is never stored: its first n doubles hold the per-row coefficients it is rebuilt from)
        CL_TRY(c, cl_diag_cg_apply_rows(a->n, a->ld, a->aval, a->rho, beta, r, a->p, Wf, a->Q, a->slab + S_PQ,
                                        a->ws, (void*)c.st));
        double pq;
        if (a->dist == nullptr) {
            CL_TRY(c, cl_diag_cg_step(a->n, a->ld, a->rho, a->Q, Wf, 0.0, qr, a->slab + S_PQ, xs, x, a->p, r,
                                      a->slab + S_QN, a->ws, (void*)c.st));
            if (!fetch(c, S_PQ, 2)) return 0;
            pq = H(c, S_PQ);
        } else {
            // row-sharded: <p, Q> is a per-rank partial until combined -- read it, take alpha
            // on the host, then update (the sequence of admm._admm_step_diag_py)
            if (!fetch(c, S_PQ, 1)) return 0;
            pq = H(c, S_PQ);
            if (isfinite(pq) && pq > 0.0) {
                CL_TRY(c, cl_diag_cg_step(a->n, a->ld, a->rho, a->Q, Wf, qr / pq, 0.0, nullptr, xs, x, a->p, r,
                                          a->slab + S_QN, a->ws, (void*)c.st));
                if (!fetch(c, S_QN, 1)) return 0;
            }
        }
        if (!isfinite(pq) || pq <= 0.0) {          // the device update was skipped
            *last_is_x = xs == x;
            *its_out = its;
            *rnorm_out = rnorm;
            *pq_bad = pq;
            return isfinite(pq) ? 2 : 1;
        }
        xs = x;
        const double qn = H(c, S_QN);
        rnorm = sqrt(qn);
        its = k + 1;
        if (rnorm <= eps) break;
        beta = qn / qr;
        qr = qn;
    }
    if (its == 0) copy(c, x, x0);
    *its_out = its;
    *rnorm_out = rnorm;
    return 0;
}

void fail(cl_admm_step_stats* out, int status, int half, int is_new, double pq) {
    out->status = status;
    out->bad_half = half;
    out->bad_is_new = is_new;
    out->pq_bad = pq;
}

}  // namespace

extern "C" int cl_admm_step_diag(const cl_admm_diag_args* a, cl_admm_step_stats* out) {
    if (a == nullptr || out == nullptr || a->n < 0 || a->ld < 2 || (a->ld & 1) || a->cg_cap < 0 ||
        a->r_v == nullptr || a->cu == nullptr)
        return CL_EARG;
    Ctx c;
    c.a = a;
    c.st = reinterpret_cast<cudaStream_t>(a->stream);
    c.rc = 0;
    c.line = 0;
    c.N = a->n * (int64_t)a->ld;
    memset(out, 0, sizeof(*out));
    out->du2 = out->dv2 = -1.0;   // the balance measures come from the one-launch step only
#define RET_RC()                \
    do {                        \
        out->err_line = c.line; \
        return c.rc;            \
    } while (0)

    // constraint values at the step start (AdmmState.constraint_values) and the primal measure
    if (!a->ax_valid)
        CL_TRY(c, cl_diag_constraint_eval(a->n, a->aval, a->ld, a->U, a->V, nullptr, nullptr, a->ax, nullptr, nullptr,
                                          nullptr, (void*)c.st));
    double pn2 = a->pnorm2_known;
    if (!(pn2 >= 0.0)) {
        const double* in[2] = {a->ax, a->b};
        const double cf[2] = {1.0, -1.0};
        lincomb(c, a->res, 2, in, cf, a->n, S_PM, true);
        if (!fetch(c, S_PM, 1)) RET_RC();
        pn2 = H(c, S_PM);
    }
    const double pmeas = sqrt(pn2) / (1.0 + a->binf);
    // Python's max/min semantics, NaN included: rel = max(floor, min(1e-2, coeff * pmeas))
    const double y = a->primal_coeff * pmeas;
    const double mn = (y < 1e-2) ? y : 1e-2;
    const double rel = (mn > a->rel_floor) ? mn : a->rel_floor;
    {
        const double* in[2] = {a->b, a->lam};
        const double cf[2] = {a->rho, -1.0};
        lincomb(c, a->nlam, 2, in, cf, a->n, -1, false);    // nlam = rho b - lam (HalfStep.rhs)
    }

    // U start; at small n also the V start and the step end, speculatively assuming U (then V)
    // is kept, read at one synchronize
    const bool spec = c.N <= SPEC_MAX_ELEMS && a->dist == nullptr;
    cg_init(c, a->U, a->V, a->r, S_RHSU, nullptr);
    if (spec) {
        cg_init(c, a->V, a->U, a->r_v, S_RHSV, a->cu);
        step_end(c, a->U, a->V);
        if (!fetch(c, S_RHSU, S_END - S_RHSU)) RET_RC();
    } else if (!fetch(c, S_RHSU, 2)) {
        RET_RC();
    }
    int last_is_x = 0;
    double pqb = 0.0;

    // U half-solve (admm.py:151-157)
    out->eps_u = pymax_tiny(rel * sqrt(H(c, S_RHSU)));
    double qr = H(c, S_R0U);
    out->res_u = sqrt(qr);
    const bool u_kept = out->res_u <= out->eps_u;
    if (!u_kept) {
        const int s = cg_loop(c, a->U, a->U_new, a->V, a->r, out->eps_u, qr, &out->it_u, &out->res_u, &last_is_x,
                              &pqb);
        if (c.rc) RET_RC();
        if (s) {
            fail(out, s, 0, last_is_x, pqb);
            return CL_OK;
        }
        selfdot(c, a->U_new, S_XXU);
        cg_init(c, a->V, a->U_new, a->r_v, S_RHSV, a->cu);       // the speculative V start used the old U
        if (!fetch(c, S_XXU, S_END - S_XXU)) RET_RC();
        if (!isfinite(H(c, S_XXU))) {                    // U's iterate is not finite
            fail(out, 3, 0, 1, 0.0);
            return CL_OK;
        }
    } else if (!spec) {
        cg_init(c, a->V, a->U, a->r_v, S_RHSV, a->cu);
        if (!fetch(c, S_RHSV, 2)) RET_RC();
    }
    out->u_reused = u_kept;
    const double* Uc = u_kept ? a->U : a->U_new;

    // V half-solve against the new U (admm.py:159-163)
    out->eps_v = pymax_tiny(rel * sqrt(H(c, S_RHSV)));
    qr = H(c, S_R0V);
    out->res_v = sqrt(qr);
    const bool v_kept = out->res_v <= out->eps_v;
    if (!v_kept) {
        const int s = cg_loop(c, a->V, a->V_new, Uc, a->r_v, out->eps_v, qr, &out->it_v, &out->res_v, &last_is_x,
                              &pqb);
        if (c.rc) RET_RC();
        if (s) {
            fail(out, s, 1, last_is_x, pqb);
            return CL_OK;
        }
        selfdot(c, a->V_new, S_XXV);
    }
    out->v_reused = v_kept;
    const double* Vc = v_kept ? a->V : a->V_new;

    // step end (admm.py:165-166 and the gap inputs of admm.py:212-217), written out of place
    // into ax / lam_new so that a non-finite V leaves the multiplier untouched
    if (!(u_kept && v_kept && spec)) {
        step_end(c, Uc, Vc);
        if (!fetch(c, S_XXV, S_E0 + 3 - S_XXV)) RET_RC();
        if (!v_kept && !isfinite(H(c, S_XXV))) {
            fail(out, 3, 1, 1, 0.0);
            return CL_OK;
        }
    }
    out->objective = H(c, S_E0);
    out->pnorm2 = H(c, S_E0 + 1);
    out->lam_b = H(c, S_E0 + 2);
    out->hit_cap = (out->it_u >= a->cg_cap && out->res_u > out->eps_u) ||
                   (out->it_v >= a->cg_cap && out->res_v > out->eps_v);
    out->err_line = c.line;
    return c.rc;
#undef RET_RC
}

// ---------------------------------------------------------------------------
// general constraints (cl_admm_step_generic): admm.admm_step's generic branch
// ---------------------------------------------------------------------------

namespace {

struct GCtx {
    const cl_admm_generic_args* a;
    cudaStream_t st;
    int rc;
    int64_t N;   // n * ld
    int line;
};

// slots inside the caller's slab
enum { G_PM = 0, G_RHSU = 1, G_RHSV = 2, G_QR = 3, G_PQ = 4, G_QN = 5, G_XX = 6, G_SCR = 7 };

bool gfetch(GCtx& c, int lo, int cnt) {
    if (c.rc) return false;
    cudaError_t e = cudaMemcpyAsync(c.a->host + lo, c.a->slab + lo, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                                    c.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.st);
    if (e != cudaSuccess) {
        c.rc = (int)e;
        c.line = __LINE__;
        return false;
    }
    return true;
}

// cl_lincomb in mode PAIRS with at most one dot (da, db); dot_slot < 0: none
void glin(GCtx& c, double* out, int nin, const double* const* in, const double* coef, int64_t N, int dot_slot,
          uint8_t da = CL_OUT, uint8_t db = CL_OUT) {
    cl_lincomb_args L;
    memset(&L, 0, sizeof(L));
    L.nin = nin;
    L.mode = CL_DOT_PAIRS;
    for (int j = 0; j < nin; ++j) {
        L.in[j] = in[j];
        L.coef[j] = coef[j];
    }
    L.out = out;
    if (dot_slot >= 0) {
        L.ndot = 1;
        L.da[0] = da;
        L.db[0] = db;
    }
    CL_TRY(c, cl_lincomb(&L, N, dot_slot >= 0 ? c.a->slab + dot_slot : nullptr, c.a->ws, (void*)c.st));
}

void gconstraint(GCtx& c, const double* X, const double* Y, double* out) {
    const cl_admm_generic_args* a = c.a;
    CL_TRY(c, cl_constraint_eval(a->m, a->con_indptr, a->con_pi, a->con_pj, a->con_val, a->ld, X, Y, nullptr, nullptr,
                                 out, nullptr, nullptr, nullptr, (void*)c.st));
}

bool single_entry(const cl_admm_generic_args* a) { return a->single_a != nullptr && a->ld <= 64; }

// HalfStep.apply: out = rho (A*(A(W Wf^T)) Wf + W); <W, out> -> slab[dot_slot] (dot_slot < 0: none)
void gapply(GCtx& c, const double* W, const double* Wf, double* out, int dot_slot) {
    const cl_admm_generic_args* a = c.a;
    if (single_entry(a)) {
        CL_TRY(c, cl_single_entry_apply(a->apat.nrows, a->apat.indptr, a->apat.indices, a->single_a, a->ld, W, Wf,
                                        a->rho, out, a->slab + (dot_slot >= 0 ? dot_slot : G_SCR), a->ws,
                                        (void*)c.st));
        return;
    }
    gconstraint(c, W, Wf, a->y);
    cl_pattern P = a->apat;
    P.cv = nullptr;
    P.c_coeff = 0.0;
    P.w1 = a->y;
    P.w2 = nullptr;
    cl_epilogue E;
    memset(&E, 0, sizeof(E));
    E.ny = 1;
    E.Y[0] = W;
    E.ycoef[0] = a->rho;
    if (dot_slot >= 0) {
        E.ndot = 1;
        E.da[0] = 0;        // Y[0] = W
        E.db[0] = CL_OUT;
    }
    CL_TRY(c, cl_pattern_spmm(&P, Wf, a->ld, a->rho, &E, out, dot_slot >= 0 ? a->slab + dot_slot : nullptr,
                              dot_slot >= 0 ? a->ws : nullptr, (void*)c.st));
}

// HalfStep.rhs: out = S_b Wf + rho Wf, S_b = -scale C - A*(lam) + rho A*(b); ||out||^2 -> slab[slot]
void grhs(GCtx& c, const double* Wf, double* out, int slot) {
    const cl_admm_generic_args* a = c.a;
    {
        const double* in[1] = {a->lam};
        const double cf[1] = {-1.0};
        glin(c, a->nlam, 1, in, cf, a->m, -1);
    }
    {
        const double* in[1] = {a->b};
        const double cf[1] = {a->rho};
        glin(c, a->rhob, 1, in, cf, a->m, -1);
    }
    cl_pattern P = a->omega;
    P.c_coeff = -a->scale;
    P.w1 = a->nlam;
    P.w2 = a->rhob;
    cl_epilogue E;
    memset(&E, 0, sizeof(E));
    E.ny = 1;
    E.Y[0] = Wf;
    E.ycoef[0] = a->rho;
    E.ndot = 1;
    E.da[0] = CL_OUT;
    E.db[0] = CL_OUT;
    CL_TRY(c, cl_pattern_spmm(&P, Wf, a->ld, 1.0, &E, out, a->slab + slot, a->ws, (void*)c.st));
}

// HalfStep.cg (admm.py:65): x = x0, then CG on the half-step operator. Returns 0, or the
// failure status (1 non-finite curvature, 2 non-positive curvature, 3 non-finite iterate).
int gcg(GCtx& c, double* x, const double* x0, const double* Wf, const double* rhs, double eps, int* its_out,
        double* rnorm_out, double* pq_bad) {
    const cl_admm_generic_args* a = c.a;
    int its = 0;
    {
        const double* in[1] = {x0};
        const double cf[1] = {1.0};
        glin(c, x, 1, in, cf, c.N, -1);
    }
    gapply(c, x, Wf, a->Q, -1);
    {
        const double* in[2] = {rhs, a->Q};
        const double cf[2] = {1.0, -1.0};
        glin(c, a->r, 2, in, cf, c.N, G_QR);
    }
    if (!gfetch(c, G_QR, 1)) return 0;
    double qr = a->host[G_QR];
    double rnorm = sqrt(qr);
    *its_out = 0;
    *rnorm_out = rnorm;
    if (rnorm <= eps) return 0;
    {
        const double* in[1] = {a->r};
        const double cf[1] = {1.0};
        glin(c, a->p, 1, in, cf, c.N, -1);
    }
    const bool pair = a->pair != nullptr && single_entry(a);
    if (pair) {
        CL_TRY(c, cl_pair_pack(a->n, a->ld, Wf, a->pair, 1, (void*)c.st));
        CL_TRY(c, cl_pair_pack(a->n, a->ld, a->p, a->pair, 0, (void*)c.st));
    }
    for (int k = 0; k < a->cg_cap; ++k) {
        if (pair)
            CL_TRY(c, cl_single_entry_apply_pair(a->apat.nrows, a->apat.indptr, a->apat.indices, a->single_a, a->ld,
                                                 a->pair, a->rho, a->Q, a->slab + G_PQ, a->ws, (void*)c.st));
        else
            gapply(c, a->p, Wf, a->Q, G_PQ);
        CL_TRY(c, cl_cg_step_dev(c.N, qr, a->slab + G_PQ, x, x, a->p, a->r, a->Q, a->slab + G_QN, a->ws,
                                 (void*)c.st));
        if (!gfetch(c, G_PQ, 2)) return 0;
        const double pq = a->host[G_PQ];
        if (!isfinite(pq)) {
            *pq_bad = pq;
            *its_out = its;
            return 1;
        }
        if (pq <= 0.0) {
            *pq_bad = pq;
            *its_out = its;
            return 2;
        }
        const double qn = a->host[G_QN];
        rnorm = sqrt(qn);
        its = k + 1;
        if (rnorm <= eps) break;
        if (pair) {
            CL_TRY(c, cl_cg_direction_pair(a->n, a->ld, qn / qr, a->r, a->p, a->pair, (void*)c.st));
        } else {
            const double* in[2] = {a->r, a->p};
            const double cf[2] = {1.0, qn / qr};
            glin(c, a->p, 2, in, cf, c.N, -1);
        }
        qr = qn;
    }
    {
        const double* in[1] = {x};
        const double cf[1] = {0.0};
        glin(c, nullptr, 1, in, cf, c.N, G_XX, 0, 0);
    }
    *its_out = its;
    *rnorm_out = rnorm;
    if (!gfetch(c, G_XX, 1)) return 0;
    if (!isfinite(a->host[G_XX])) return 3;
    return 0;
}

}  // namespace

extern "C" int cl_admm_step_generic(const cl_admm_generic_args* a, cl_admm_step_stats* out) {
    if (a == nullptr || out == nullptr || a->n < 0 || a->m < 0 || a->ld < 2 || (a->ld & 1) || a->cg_cap < 0 ||
        a->ax_new == nullptr || a->U_new == nullptr || a->V_new == nullptr || a->omega.indptr == nullptr ||
        a->apat.indptr == nullptr)
        return CL_EARG;
    GCtx c;
    c.a = a;
    c.st = reinterpret_cast<cudaStream_t>(a->stream);
    c.rc = 0;
    c.line = 0;
    c.N = a->n * (int64_t)a->ld;
    memset(out, 0, sizeof(*out));
    out->du2 = out->dv2 = -1.0;
#define GRET()                  \
    do {                        \
        out->err_line = c.line; \
        return c.rc;            \
    } while (0)
    const double* ax = a->ax;
    if (ax == nullptr) {
        gconstraint(c, a->U, a->V, a->ax_new);
        ax = a->ax_new;
    }
    {
        const double* in[2] = {ax, a->b};
        const double cf[2] = {1.0, -1.0};
        glin(c, a->y, 2, in, cf, a->m, G_PM);
    }
    if (!gfetch(c, G_PM, 1)) GRET();
    const double pmeas = sqrt(a->host[G_PM]) / (1.0 + a->binf);
    const double yv = a->primal_coeff * pmeas;
    const double mn = (yv < 1e-2) ? yv : 1e-2;
    const double rel = (mn > a->rel_floor) ? mn : a->rel_floor;
    double pqb = 0.0;

    grhs(c, a->V, a->rhs, G_RHSU);
    if (!gfetch(c, G_RHSU, 1)) GRET();
    out->eps_u = pymax_tiny(rel * sqrt(a->host[G_RHSU]));
    int s = gcg(c, a->U_new, a->U, a->V, a->rhs, out->eps_u, &out->it_u, &out->res_u, &pqb);
    if (c.rc) GRET();
    if (s) {
        fail(out, s, 0, 1, pqb);
        GRET();
    }
    grhs(c, a->U_new, a->rhs, G_RHSV);
    if (!gfetch(c, G_RHSV, 1)) GRET();
    out->eps_v = pymax_tiny(rel * sqrt(a->host[G_RHSV]));
    s = gcg(c, a->V_new, a->V, a->U_new, a->rhs, out->eps_v, &out->it_v, &out->res_v, &pqb);
    if (c.rc) GRET();
    if (s) {
        fail(out, s, 1, 1, pqb);
        GRET();
    }
    gconstraint(c, a->U_new, a->V_new, a->ax_new);
    {
        const double* in[2] = {a->ax_new, a->b};
        const double cf[2] = {1.0, -1.0};
        glin(c, a->y, 2, in, cf, a->m, G_PM);
    }
    {
        const double* in[2] = {a->lam, a->y};
        const double cf[2] = {1.0, a->rho};
        glin(c, a->lam, 2, in, cf, a->m, -1);
    }
    if (!gfetch(c, G_PM, 1)) GRET();
    out->pnorm2 = a->host[G_PM];
    out->hit_cap = (out->it_u >= a->cg_cap && out->res_u > out->eps_u) ||
                   (out->it_v >= a->cg_cap && out->res_v > out->eps_v);
    GRET();
#undef GRET
}

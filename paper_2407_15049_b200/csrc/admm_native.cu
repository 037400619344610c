// admm_native.cu -- one ADMM step (admm.py:136 admm_step) for diagonal
// constraints, driven from native host code.
//
// The Python host (admm.py) issues the same launches with a Python-side
// decision after each reduction; at small n that host round trip, not the
// GPU, bounds the step rate. This file runs the identical sequence of
// launches and scalar decisions in C++: the CG stop test, alpha/beta, the
// curvature and finiteness checks of cg_solve (admm.py:65), the tolerance
// schedule and the dual ascent. Each decision point is one pinned 8-byte
// read after a stream synchronize. The kernels and their order are exactly
// those of the Python path (HalfStep.rhs / HalfStep._cg_diag / admm_step),
// so both paths produce bit-identical iterates
// (tests/test_gpu_admm_native.py).

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "culorads.h"

namespace {

struct Ctx {
    const cl_admm_diag_args* a;
    cudaStream_t st;
    int rc;
    int64_t N;   // n * ld
    int line;    // source line of the first failing call (diagnostics)
};

#define CL_TRY(c, expr)                 \
    do {                                \
        if (!(c).rc) {                  \
            (c).rc = (expr);            \
            if ((c).rc) (c).line = __LINE__; \
        }                               \
    } while (0)

// Reduction slots inside the caller's slab. The values read together at one
// decision point are contiguous, so each decision costs one synchronize.
enum { S_PM = 0, S_RHS = 1, S_R0 = 2, S_XXU = 3, S_PQ = 4, S_QN = 5, S_PN = 6, S_XXV = 7, S_OBJ = 8, S_LB = 9,
       S_E0 = 10 };   // S_E0..S_E0+2: the fused step-end dots (objective, ||ax-b||^2, lam_new.b)

// ld <= FUSED_LD: the rhs + initial residual and the step end run as single fused SpMM passes
// (any ld: the fused epilogues reduce the row dot over all column chunks)
constexpr int FUSED_LD = 1 << 30;

// Copy slab[lo, lo+cnt) to the pinned host buffer and wait.
bool fetch(Ctx& c, int lo, int cnt) {
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

double H(const Ctx& c, int slot) { return c.a->host[slot]; }

void lincomb(Ctx& c, double* out, int nin, const double* const* in, const double* coef, int64_t N, int dot_slot,
             bool dot_out_out) {
    if (c.rc) return;
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
    if (c.rc) return;
    cl_lincomb_args L;
    memset(&L, 0, sizeof(L));
    L.nin = 1;
    L.mode = CL_DOT_PAIRS;
    L.in[0] = x;
    L.coef[0] = 0.0;
    L.ndot = 1;
    CL_TRY(c, cl_lincomb(&L, c.N, c.a->slab + slot, c.a->ws, (void*)c.st));
}

// rhs = S_b Wf + rho Wf, S_b = -scale C + diag(a (rho b - lam))  (HalfStep.rhs, diagonal branch);
// nlam = rho b - lam is computed once per step (lam does not change inside it).
void rhs(Ctx& c, const double* Wf) {
    const cl_admm_diag_args* a = c.a;
    if (c.rc) return;
    cl_pattern P = a->cpat;
    P.c_coeff = 1.0;
    cl_epilogue E;
    memset(&E, 0, sizeof(E));
    E.ny = 1;
    E.Y[0] = Wf;
    E.ycoef[0] = a->rho;
    E.ndot = 1;
    E.da[0] = CL_OUT;
    E.db[0] = CL_OUT;
    E.drow = a->nlam;
    E.dmul = a->aval;
    CL_TRY(c, cl_pattern_spmm(&P, Wf, a->ld, -a->scale, &E, a->rhs, a->slab + S_RHS, a->ws, (void*)c.st));
}

// max(v, 1e-300) with Python semantics (v is kept unless 1e-300 > v; NaN stays NaN)
double pymax_tiny(double v) { return (1e-300 > v) ? 1e-300 : v; }

// One half-step: rhs, then admm.py:65 cg_solve on the diagonal operator
// (HalfStep._cg_diag), x0 read only, result in x. The rhs norm (tolerance)
// and the initial residual are read at one synchronize, together with the
// pending finiteness test of the previous half's iterate (xx_prev_slot >= 0).
// Returns 0 ok, 1 non-finite curvature, 2 non-positive curvature,
// 4 the previous half's iterate is not finite.
int half(Ctx& c, const double* x0, double* x, const double* Wf, double rel, int xx_prev_slot, double* eps_out,
         int* its_out, double* rnorm_out, int* last_is_x, double* pq_bad, int* reused) {
    const cl_admm_diag_args* a = c.a;
    *its_out = 0;
    *last_is_x = 0;
    *reused = 0;
    if (a->ld <= FUSED_LD) {
        // rhs (never stored), Q(x0) and r = rhs - Q(x0) in one pass over C's rows
        cl_pattern P = a->cpat;
        P.c_coeff = 1.0;
        CL_TRY(c, cl_diag_admm_cg_init(&P, Wf, x0, a->ld, a->scale, a->rho, a->nlam, a->aval, a->r, a->slab + S_RHS,
                                       a->ws, (void*)c.st));
    } else {
        rhs(c, Wf);
        CL_TRY(c, cl_diag_cg_apply(a->n, a->ld, a->aval, a->rho, 0.0, nullptr, const_cast<double*>(x0), Wf, a->Q,
                                   a->slab + S_PQ, a->ws, (void*)c.st));
        const double* in[2] = {a->rhs, a->Q};
        const double cf[2] = {1.0, -1.0};
        lincomb(c, a->r, 2, in, cf, c.N, S_R0, true);
    }
    if (!fetch(c, S_RHS, xx_prev_slot >= 0 ? 3 : 2)) return 0;
    if (xx_prev_slot >= 0 && !isfinite(H(c, xx_prev_slot))) return 4;
    const double eps = pymax_tiny(rel * sqrt(H(c, S_RHS)));
    *eps_out = eps;
    double qr = H(c, S_R0);
    double rnorm = sqrt(qr);
    *rnorm_out = rnorm;
    if (rnorm <= eps) {
        *reused = 1;          // the iterate stays x0: no copy, the caller keeps x0 as the new factor
        return 0;
    }
    int its = 0;
    double beta = 0.0;
    const double* xs = x0;
    for (int k = 0; k < a->cg_cap; ++k) {
        CL_TRY(c, cl_diag_cg_apply(a->n, a->ld, a->aval, a->rho, beta, a->r, a->p, Wf, a->Q, a->slab + S_PQ,
                                   a->ws, (void*)c.st));
        if (!fetch(c, S_PQ, 1)) return 0;
        const double pq = H(c, S_PQ);
        if (!isfinite(pq) || pq <= 0.0) {
            *last_is_x = xs == x;
            *its_out = its;
            *pq_bad = pq;
            return isfinite(pq) ? 2 : 1;
        }
        const double alpha = qr / pq;
        CL_TRY(c, cl_cg_step(c.N, alpha, xs, x, a->p, a->r, a->Q, a->slab + S_QN, a->ws, (void*)c.st));
        xs = x;
        if (!fetch(c, S_QN, 1)) return 0;
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

}  // namespace

extern "C" int cl_admm_step_diag(const cl_admm_diag_args* a, cl_admm_step_stats* out) {
    if (a == nullptr || out == nullptr || a->n < 0 || a->ld < 2 || (a->ld & 1) || a->cg_cap < 0) return CL_EARG;
    Ctx c;
    c.a = a;
    c.st = reinterpret_cast<cudaStream_t>(a->stream);
    c.rc = 0;
    c.line = 0;
    c.N = a->n * (int64_t)a->ld;
    memset(out, 0, sizeof(*out));

    // constraint values at the step start (AdmmState.constraint_values) and the primal measure
    if (!a->ax_valid)
        CL_TRY(c, cl_diag_constraint_eval(a->n, a->aval, a->ld, a->U, a->V, nullptr, nullptr, a->ax, nullptr, nullptr,
                                          nullptr, (void*)c.st));
    double pn2 = a->pnorm2_known;
    if (!(pn2 >= 0.0)) {
        const double* in[2] = {a->ax, a->b};
        const double cf[2] = {1.0, -1.0};
        lincomb(c, a->res, 2, in, cf, a->n, S_PM, true);
        if (!fetch(c, S_PM, 1)) { out->err_line = c.line; return c.rc; }
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
        lincomb(c, a->nlam, 2, in, cf, a->n, -1, false);
    }

    // U half-solve, then V half-solve against the new U (admm.py:151-163)
    int last_is_x = 0, reused = 0;
    double pqb = 0.0;
    int s = half(c, a->U, a->U_new, a->V, rel, -1, &out->eps_u, &out->it_u, &out->res_u, &last_is_x, &pqb, &reused);
    if (c.rc) { out->err_line = c.line; return c.rc; }
    if (s) {
        out->status = s;
        out->bad_half = 0;
        out->bad_is_new = last_is_x;
        out->pq_bad = pqb;
        return CL_OK;
    }
    out->u_reused = reused;
    const double* Uc = reused ? a->U : a->U_new;
    if (!reused) selfdot(c, a->U_new, S_XXU);
    s = half(c, a->V, a->V_new, Uc, rel, reused ? -1 : S_XXU, &out->eps_v, &out->it_v, &out->res_v, &last_is_x, &pqb,
             &reused);
    if (c.rc) { out->err_line = c.line; return c.rc; }
    if (s == 4) {                      // U's iterate was not finite (checked one synchronize late)
        out->status = 3;
        out->bad_half = 0;
        out->bad_is_new = 1;
        return CL_OK;
    }
    if (s) {
        out->status = s;
        out->bad_half = 1;
        out->bad_is_new = last_is_x;
        out->pq_bad = pqb;
        return CL_OK;
    }
    out->v_reused = reused;
    const double* Vc = reused ? a->V : a->V_new;
    if (!reused) selfdot(c, a->V_new, S_XXV);

    // dual ascent on the new constraint values (admm.py:165-166), written out of place into
    // lam_new so that a late-detected non-finite V leaves the multiplier untouched; then the
    // objective <C V, U> and lam_new . b that admm_run's gap test reads (admm.py:212-217)
    if (a->ld <= FUSED_LD) {
        cl_pattern P = a->cpat;
        P.c_coeff = 1.0;
        CL_TRY(c, cl_diag_admm_step_end(&P, Uc, Vc, a->ld, a->aval, a->b, a->lam, a->rho, a->ax, a->lam_new,
                                        a->slab + S_E0, a->ws, (void*)c.st));
        if (!fetch(c, S_XXV, S_E0 + 3 - S_XXV)) { out->err_line = c.line; return c.rc; }
        if (!out->v_reused && !isfinite(H(c, S_XXV))) {
            out->status = 3;
            out->bad_half = 1;
            out->bad_is_new = 1;
            return CL_OK;
        }
        out->objective = H(c, S_E0);
        out->pnorm2 = H(c, S_E0 + 1);
        out->lam_b = H(c, S_E0 + 2);
    } else {
        CL_TRY(c, cl_diag_constraint_eval(a->n, a->aval, a->ld, Uc, Vc, nullptr, nullptr, a->ax, nullptr, nullptr,
                                          nullptr, (void*)c.st));
        {
            const double* in[2] = {a->ax, a->b};
            const double cf[2] = {1.0, -1.0};
            lincomb(c, a->res, 2, in, cf, a->n, S_PN, true);
        }
        {
            const double* in[2] = {a->lam, a->res};
            const double cf[2] = {1.0, a->rho};
            lincomb(c, a->lam_new, 2, in, cf, a->n, -1, false);
        }
        if (!c.rc) {
            cl_pattern P = a->cpat;
            P.c_coeff = 1.0;
            cl_epilogue E;
            memset(&E, 0, sizeof(E));
            E.nz = 1;
            E.Z[0] = Uc;
            E.ndot = 1;
            E.da[0] = CL_OUT;
            E.db[0] = 16;
            CL_TRY(c, cl_pattern_spmm(&P, Vc, a->ld, 1.0, &E, nullptr, a->slab + S_OBJ, a->ws, (void*)c.st));
        }
        if (!c.rc) {
            cl_lincomb_args L;
            memset(&L, 0, sizeof(L));
            L.nin = 2;
            L.mode = CL_DOT_PAIRS;
            L.in[0] = a->lam_new;
            L.in[1] = a->b;
            L.ndot = 1;
            L.da[0] = 0;
            L.db[0] = 1;
            CL_TRY(c, cl_lincomb(&L, a->n, a->slab + S_LB, a->ws, (void*)c.st));
        }
        if (!fetch(c, S_PN, 4)) { out->err_line = c.line; return c.rc; }
        if (!out->v_reused && !isfinite(H(c, S_XXV))) {
            out->status = 3;
            out->bad_half = 1;
            out->bad_is_new = 1;
            return CL_OK;
        }
        out->pnorm2 = H(c, S_PN);
        out->objective = H(c, S_OBJ);
        out->lam_b = H(c, S_LB);
    }
    out->hit_cap = (out->it_u >= a->cg_cap && out->res_u > out->eps_u) ||
                   (out->it_v >= a->cg_cap && out->res_v > out->eps_v);
    out->err_line = c.line;
    return c.rc;
}

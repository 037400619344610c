// alm_native.cu -- the ALM inner solve (alm.py:268 alm_inner) for diagonal
// constraints, driven from native host code.
//
// Same launches, in the same order, with the same operands as the Python host
// path (alm.py _inner / AlmCore / lbfgs_direction / best_step); the host-side
// scalar algebra -- the vector-free two-loop recursion over the Gram matrix,
// the quartic line-search coefficients, the cubic roots and the tie-breaking
// of best_step (alm.py:166/202), the curvature-pair bookkeeping -- is
// restated here operation for operation, so the iterates are bit-identical
// to the Python-driven path (tests/test_gpu_alm_native.py). Each iteration
// needs two pinned reads: the direction's Gram row travels with the
// line-search scalars, then the update's reductions.

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <time.h>

#include "culorads.h"

namespace {

constexpr int MAXB = CL_ALM_MAXBUF;

struct Ctx {
    const cl_alm_inner_args* a;
    cudaStream_t st;
    int rc;
    int line;
    int64_t N;
    bool generic;    // general constraints (cl_alm_inner_generic)
    int64_t M;       // m-vector length
};

#define TRY(c, expr)                      \
    do {                                  \
        if (!(c).rc) {                    \
            (c).rc = (expr);              \
            if ((c).rc) (c).line = __LINE__; \
        }                                 \
    } while (0)

// slab layout of the Python path (AlmCore.S_*): direction dots at 0, line search at 40/48, update at 64
enum { S_DIR = 0, S_LS = 40, S_MV = 48, S_UPD = 64 };

bool fetch(Ctx& c, int count) {
    if (c.rc) return false;
    if (c.a->dist != nullptr) {     // row-sharded: the partial sums are combined over the ranks
        const int rc = c.a->dist->reduce(c.a->dist->ctx, c.a->slab, c.a->host, count, (void*)c.st);
        if (rc != 0) {
            c.rc = CL_EARG;
            c.line = __LINE__;
            return false;
        }
        return true;
    }
    cudaError_t e = cudaMemcpyAsync(c.a->host, c.a->slab, count * sizeof(double), cudaMemcpyDeviceToHost, c.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.st);
    if (e != cudaSuccess) {
        c.rc = (int)e;
        c.line = __LINE__;
        return false;
    }
    return true;
}

double now_s() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);   // the clock of Python's time.perf_counter on Linux
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

// ---------------------------------------------------------------------------
// L-BFGS history: pairs of buffer indices, Gram matrix over buffer indices
// ---------------------------------------------------------------------------

struct Pair {
    int d, y;
    double sigma, beta;
};

struct Hist {
    int cap = 0, cnt = 0, head = 0;   // ring, oldest at head
    Pair p[CL_ALM_MAXMEM];
    double G[MAXB][MAXB];
    const Pair& at(int k) const { return p[(head + k) % CL_ALM_MAXMEM]; }
    void set(int i, int j, double v) {
        G[i][j] = v;
        G[j][i] = v;
    }
};

// Pool of factor buffers (alm.py FactorPool semantics: LIFO free list)
struct Pool {
    int free_[MAXB];
    int nfree = 0;
    int get() { return nfree > 0 ? free_[--nfree] : -1; }
    void put(int b) { free_[nfree++] = b; }
};

// alm.py:166 _real_cubic_roots (+ two Newton polish steps), as in alm.cubic_roots
int cubic_roots(double c3, double c2, double c1, double c0, double* out) {
    const double b2 = c2 / c3, b1 = c1 / c3, b0 = c0 / c3;
    const double shift = b2 / 3.0;
    const double P = b1 - b2 * b2 / 3.0;
    const double Q = b0 - b2 * b1 / 3.0 + 2.0 * pow(b2, 3.0) / 27.0;
    double ts[3];
    int nt;
    if (fabs(P) < 1e-300 && fabs(Q) < 1e-300) {
        ts[0] = 0.0;
        nt = 1;
    } else if (-4.0 * pow(P, 3.0) - 27.0 * pow(Q, 2.0) > 0.0) {
        const double amp = 2.0 * sqrt(-P / 3.0);
        const double phase = acos(fmin(1.0, fmax(-1.0, 3.0 * Q / (P * amp)))) / 3.0;
        for (int k = 0; k < 3; ++k) ts[k] = amp * cos(phase - 2.0 * M_PI * k / 3.0);
        nt = 3;
    } else {
        const double h = -0.5 * Q;
        const double rad = sqrt(fmax(0.0, Q * Q / 4.0 + pow(P, 3.0) / 27.0));
        ts[0] = copysign(pow(fabs(h + rad), 1.0 / 3.0), h + rad) + copysign(pow(fabs(h - rad), 1.0 / 3.0), h - rad);
        nt = 1;
    }
    for (int k = 0; k < nt; ++k) {
        double x = ts[k] - shift;
        for (int it = 0; it < 2; ++it) {
            const double f = ((c3 * x + c2) * x + c1) * x + c0;
            const double df = (3.0 * c3 * x + 2.0 * c2) * x + c1;
            if (df != 0.0 && isfinite(f) && isfinite(df)) x -= f / df;
        }
        out[k] = x;
    }
    return nt;
}

double qval(const double* a, double t) { return ((a[0] * t + a[1]) * t + a[2]) * t * t + a[3] * t; }

// alm.py:202 best_step: global minimiser of the ray quartic; returns zero_direction
bool best_step(const double* a, double* tau) {
    const double a1 = a[0], a2 = a[1], a3 = a[2], a4 = a[3];
    if (a1 == 0.0 && a2 == 0.0 && a3 == 0.0 && a4 == 0.0) {
        *tau = 0.0;
        return true;
    }
    double cand[4];
    int nc = 0;
    if (a1 != 0.0) {
        nc = cubic_roots(4.0 * a1, 3.0 * a2, 2.0 * a3, a4, cand);
        cand[nc++] = 0.0;
    } else if (a2 != 0.0) {
        cand[nc++] = 0.0;
        const double disc = a3 * a3 - 3.0 * a2 * a4;
        if (disc >= 0.0) {
            const double sg[2] = {1.0, -1.0};
            for (int k = 0; k < 2; ++k) {
                const double t = (-a3 + sg[k] * sqrt(disc)) / (3.0 * a2);
                if (6.0 * a2 * t + 2.0 * a3 > 0.0) cand[nc++] = t;
            }
        }
    } else if (a3 != 0.0) {
        cand[nc++] = a3 > 0.0 ? -a4 / (2.0 * a3) : 0.0;
    } else {
        cand[nc++] = 0.0;
    }
    double vals[4];
    double vmin = INFINITY;
    for (int k = 0; k < nc; ++k) {
        vals[k] = isfinite(cand[k]) ? qval(a, cand[k]) : INFINITY;
        // Python min(): the first minimum wins, NaN never replaces
        if (k == 0 || vals[k] < vmin) vmin = vals[k];
    }
    const double band = vmin + 1e-12 * (1.0 + fabs(vmin));
    // min over tied candidates with key (|t|, -t): first minimal key wins
    bool have = false;
    double best = 0.0;
    for (int k = 0; k < nc; ++k) {
        if (!(vals[k] <= band)) continue;
        const double t = cand[k];
        if (!have || fabs(t) < fabs(best) || (fabs(t) == fabs(best) && -t < -best)) {
            best = t;
            have = true;
        }
    }
    *tau = best;
    return false;
}

double* B(const Ctx& c, int i) { return c.a->bufs[i]; }

// AlmCore.grad_value, diagonal branch: one cl_diag_alm_update launch + one fetch
void lincomb_n(Ctx& c, double* out, int nin, const double* const* in, const double* coef, int64_t N, double* slab,
               int mode, int ndot, const uint8_t* da, const uint8_t* db) {
    cl_lincomb_args L;
    memset(&L, 0, sizeof(L));
    L.nin = nin;
    L.mode = mode;
    for (int j = 0; j < nin; ++j) {
        L.in[j] = in[j];
        L.coef[j] = coef[j];
    }
    L.out = out;
    L.ndot = ndot;
    for (int k = 0; k < ndot && da != nullptr; ++k) {
        L.da[k] = da[k];
        L.db[k] = db[k];
    }
    TRY(c, cl_lincomb(&L, N, ndot ? slab : nullptr, ndot ? c.a->ws : nullptr, (void*)c.st));
}

// AlmCore.grad_value, generic branch (alm.py AlmCore.grad_value): the step (unless refresh),
// res = ax - b with rr, lam.res; <CR, R>; w = lam + rho res; g = 2 A*(w) R + 2 scale C R over
// Omega_A; y = g - g_old; the Gram rows of g and y; one fetch. Results in the diagonal
// branch's layout s[0..]: crr, gg, yd, lres, rr, yy, gy, gH[], yH[].
bool grad_value_generic(Ctx& c, double* R, const double* gold, double* gnew, double* y, const double* const* H, int nh,
                        const double* D, const double* CD, double tau, bool refresh, const double* ax_in,
                        double* ax_out, double* s) {
    const cl_alm_inner_args* a = c.a;
    const double* ax = ax_in;
    if (!refresh) {
        const double* i1[2] = {R, D};
        const double c1[2] = {1.0, tau};
        lincomb_n(c, R, 2, i1, c1, c.N, nullptr, CL_DOT_PAIRS, 0, nullptr, nullptr);
        const double* i2[2] = {a->CR, CD};
        lincomb_n(c, a->CR, 2, i2, c1, c.N, nullptr, CL_DOT_PAIRS, 0, nullptr, nullptr);
        const double* i3[3] = {ax_in, a->q1, a->q2};
        const double c3[3] = {1.0, tau, tau * tau};
        lincomb_n(c, ax_out, 3, i3, c3, c.M, nullptr, CL_DOT_PAIRS, 0, nullptr, nullptr);
        ax = ax_out;
    }
    {
        const double* in[3] = {ax, a->b, a->lam};
        const double cf[3] = {1.0, -1.0, 0.0};
        const uint8_t da[2] = {CL_OUT, 2}, db[2] = {CL_OUT, CL_OUT};
        lincomb_n(c, a->res, 3, in, cf, c.M, a->slab + S_UPD + 4, CL_DOT_PAIRS, 2, da, db);   // rr, lam.res
    }
    {
        const double* in[2] = {a->CR, R};
        const double cf[2] = {0.0, 0.0};
        const uint8_t da[1] = {0}, db[1] = {1};
        lincomb_n(c, nullptr, 2, in, cf, c.N, a->slab + S_UPD, CL_DOT_PAIRS, 1, da, db);       // <CR, R>
    }
    {
        const double* in[2] = {a->lam, a->res};
        const double cf[2] = {1.0, a->rho};
        lincomb_n(c, a->wv, 2, in, cf, c.M, nullptr, CL_DOT_PAIRS, 0, nullptr, nullptr);   // w = lam + rho res
    }
    {
        cl_pattern P = a->apat;
        P.cv = nullptr;
        P.c_coeff = 0.0;
        P.w1 = a->wv;
        P.w2 = nullptr;
        cl_epilogue E;
        memset(&E, 0, sizeof(E));
        E.ny = 1;
        E.Y[0] = a->CR;
        E.ycoef[0] = 2.0 * a->scale;
        TRY(c, cl_pattern_spmm(&P, R, a->ld, 2.0, &E, gnew, nullptr, nullptr, (void*)c.st));
    }
    {
        const double* in[2] = {gnew, gold};
        const double cf[2] = {1.0, -1.0};
        lincomb_n(c, y, 2, in, cf, c.N, nullptr, CL_DOT_PAIRS, 0, nullptr, nullptr);
    }
    {
        const double* in[2 + 2 * CL_ALM_MAXMEM + 1];
        double cf[2 + 2 * CL_ALM_MAXMEM + 1];
        in[0] = gnew;
        in[1] = y;
        for (int k = 0; k < nh; ++k) in[2 + k] = H[k];
        for (int k = 0; k < 2 + nh; ++k) cf[k] = 0.0;
        lincomb_n(c, nullptr, 2 + nh, in, cf, c.N, a->slab + S_UPD + 8, CL_DOT_FIRST_TWO, 1, nullptr, nullptr);
    }
    if (!fetch(c, S_UPD + 8 + 2 * CL_MAXIN)) return false;
    const double* h = a->host + S_UPD;
    s[0] = h[0];
    s[1] = h[8];
    s[3] = h[5];
    s[4] = h[4];
    s[5] = h[8 + CL_MAXIN];
    s[6] = h[9];
    for (int k = 0; k < nh; ++k) {
        s[7 + k] = h[10 + k];
        s[7 + CL_MAXIN + k] = h[8 + CL_MAXIN + 1 + k];
    }
    s[2] = (D != nullptr && nh > 0 && H[nh - 1] == D) ? s[7 + CL_MAXIN + nh - 1] : 0.0;
    return true;
}

bool grad_value(Ctx& c, double* R, int g_old, const double* gold_ptr, int g_new, int ybuf, const int* H, int nh,
                const double* D, const double* CD, double tau, bool refresh, const double* ax_in, double* ax_out,
                double* s) {
    const cl_alm_inner_args* a = c.a;
    if (c.generic) {
        const double* Hp[2 * CL_ALM_MAXMEM + 1];
        for (int j = 0; j < nh; ++j) Hp[j] = c.a->bufs[H[j]];
        return grad_value_generic(c, R, g_old >= 0 ? c.a->bufs[g_old] : gold_ptr, c.a->bufs[g_new], c.a->bufs[ybuf],
                                  Hp, nh, D, CD, tau, refresh, ax_in, ax_out, s);
    }
    cl_diag_update_args u;
    memset(&u, 0, sizeof(u));
    u.n = a->n;
    u.ld = a->ld;
    u.aval = a->aval;
    u.tau = tau;
    u.rho = a->rho;
    u.scale = a->scale;
    u.R = R;
    u.D = D;
    u.CR = a->CR;
    u.CD = CD;
    u.ax = ax_in;
    u.ax_out = ax_out;
    u.q1 = a->q1;
    u.q2 = a->q2;
    u.lam = a->lam;
    u.b = a->b;
    u.g_old = g_old >= 0 ? B(c, g_old) : gold_ptr;
    u.g_new = B(c, g_new);
    u.y = B(c, ybuf);
    u.nh = nh;
    for (int j = 0; j < nh; ++j) u.H[j] = B(c, H[j]);
    u.refresh = refresh ? 1 : 0;
    TRY(c, cl_diag_alm_update(&u, a->slab + S_UPD, a->ws, (void*)c.st));
    if (!fetch(c, S_UPD + 7 + 2 * CL_MAXIN)) return false;
    for (int k = 0; k < 7 + 2 * CL_MAXIN; ++k) s[k] = a->host[S_UPD + k];
    return true;
}

void constraint_values(Ctx& c, const double* R, double* out) {
    const cl_alm_inner_args* a = c.a;
    if (c.generic) {
        TRY(c, cl_constraint_eval(a->m, a->con_indptr, a->con_pi, a->con_pj, a->con_val, a->ld, R, R, nullptr, nullptr,
                                  out, nullptr, nullptr, nullptr, (void*)c.st));
        return;
    }
    TRY(c, cl_diag_constraint_eval(a->n, a->aval, a->ld, R, R, nullptr, nullptr, out, nullptr, nullptr, nullptr,
                                   (void*)c.st));
}

// C's pattern for a product with X; a row-sharded solve first exchanges X's halo
bool c_pattern(Ctx& c, const double* X, cl_pattern* P) {
    *P = c.a->cpat;
    P->c_coeff = 1.0;
    if (c.a->dist != nullptr && !c.rc) {
        P->ghost = c.a->dist->exchange(c.a->dist->ctx, X, c.a->ld);
        P->nown = c.a->dist->nown;
        if (P->ghost == nullptr) {
            c.rc = CL_EARG;
            c.line = __LINE__;
            return false;
        }
    }
    return !c.rc;
}

// peer-memory ghosts: fence after the product that read the peers' rows (cl_dist_hooks)
void c_release(Ctx& c) {
    const cl_dist_hooks* d = c.a->dist;
    if (d == nullptr || d->release == nullptr || c.rc) return;
    if (d->release(d->ctx, (void*)c.st) != 0) {
        c.rc = CL_EARG;
        c.line = __LINE__;
    }
}

void c_times(Ctx& c, const double* X, double* out) {
    const cl_alm_inner_args* a = c.a;
    cl_pattern P;
    if (!c_pattern(c, X, &P)) return;
    TRY(c, cl_pattern_spmm(&P, X, a->ld, 1.0, nullptr, out, nullptr, nullptr, (void*)c.st));
    c_release(c);
}

int alm_inner(const cl_alm_inner_args* a, cl_alm_inner_stats* out, bool generic);

}  // namespace

extern "C" int cl_alm_inner_diag(const cl_alm_inner_args* a, cl_alm_inner_stats* out) {
    return alm_inner(a, out, false);
}

extern "C" int cl_alm_inner_generic(const cl_alm_inner_args* a, cl_alm_inner_stats* out) {
    if (a == nullptr || a->dist != nullptr || a->m < 0 || (a->m > 0 && (a->con_indptr == nullptr ||
        a->con_pi == nullptr || a->con_pj == nullptr || a->con_val == nullptr)) || a->res == nullptr ||
        a->apat.at_ptr == nullptr || a->zero_g == nullptr)
        return CL_EARG;
    return alm_inner(a, out, true);
}

namespace {

int alm_inner(const cl_alm_inner_args* a, cl_alm_inner_stats* out, bool generic) {
    if (a == nullptr || out == nullptr || a->n < 0 || a->ld < 2 || (a->ld & 1) || a->memory < 0 ||
        a->memory > CL_ALM_MAXMEM || a->nbuf < 2 * a->memory + 4 || a->nbuf > MAXB)
        return CL_EARG;
    Ctx c;
    c.a = a;
    c.st = reinterpret_cast<cudaStream_t>(a->stream);
    c.rc = 0;
    c.line = 0;
    c.N = a->n * (int64_t)a->ld;
    c.generic = generic;
    c.M = generic ? a->m : a->n;
    memset(out, 0, sizeof(*out));
    static thread_local Hist hist;
    hist.cap = a->memory;
    hist.cnt = 0;
    hist.head = 0;
    Pool pool;
    for (int i = a->nbuf - 1; i >= 0; --i) pool.put(i);
    double* R = a->R;
    double* ax_cur = a->ax;     // AlmCore.ax / AlmCore.ax2 (swapped after every stepping update)
    double* ax_alt = a->ax2;

    constraint_values(c, R, ax_cur);
    c_times(c, R, a->CR);
    int g = pool.get(), gscr = pool.get(), yscr = pool.get();
    double s[7 + 2 * CL_MAXIN];
    if (!grad_value(c, R, -1, a->zero_g, g, yscr, nullptr, 0, R, a->CR, 0.0, true, ax_cur, ax_cur, s)) {
        out->err_line = c.line;
        return c.rc;
    }
    double L = a->scale * s[0] + s[3] + 0.5 * a->rho * s[4];
    double gg = s[1];
    hist.set(g, g, gg);
    if (!(isfinite(L) && isfinite(gg))) {
        out->status = 1;
        return CL_OK;
    }
    const double gnorm0 = sqrt(gg);
    int iterations = 0;
    int nrec = 0;
    int status = 0;
    bool hit = true;
    for (int it = 0; it < a->max_iter; ++it) {
        const double gnorm = sqrt(gg);
        if (nrec < a->rec_cap) a->gnorms[nrec] = gnorm;
        out->n_gnorms = it + 1;
        if (gnorm / (1.0 + fabs(L)) <= a->tol) {
            hit = false;
            break;
        }
        if (a->reduce_factor >= 0.0 && gnorm <= a->reduce_factor * gnorm0) {
            hit = false;
            break;
        }

        // ---- direction (alm.py:98 via lbfgs_direction: coefficients over the Gram matrix) ----
        const int Dn = pool.get();
        int tb[2 * CL_ALM_MAXMEM + 1];
        double tc[2 * CL_ALM_MAXMEM + 1];
        int nt = 0;
        tb[nt] = g;
        tc[nt] = -1.0;
        ++nt;
        auto find = [&](int buf) {
            for (int k = 0; k < nt; ++k)
                if (tb[k] == buf) return k;
            return -1;
        };
        auto dotD = [&](int x) {
            double acc = 0.0;
            for (int k = 0; k < nt; ++k) acc += hist.G[x][tb[k]] * tc[k];
            return acc;
        };
        double alphas[CL_ALM_MAXMEM];
        for (int k = hist.cnt - 1, q = 0; k >= 0; --k, ++q) {
            const Pair& pr = hist.at(k);
            const double av = pr.beta * (pr.sigma * dotD(pr.d));
            int pos = find(pr.y);
            if (pos < 0) {
                tb[nt] = pr.y;
                tc[nt] = 0.0;
                pos = nt++;
            }
            tc[pos] = tc[pos] - av;
            alphas[q] = av;
        }
        for (int k = 0; k < hist.cnt; ++k) {
            const Pair& pr = hist.at(k);
            const double av = alphas[hist.cnt - 1 - k];
            const double bb = pr.beta * dotD(pr.y);
            int pos = find(pr.d);
            if (pos < 0) {
                tb[nt] = pr.d;
                tc[nt] = 0.0;
                pos = nt++;
            }
            tc[pos] = tc[pos] + (av - bb) * pr.sigma;
        }
        {
            cl_lincomb_args Lc;
            memset(&Lc, 0, sizeof(Lc));
            Lc.nin = nt;
            Lc.mode = CL_DOT_OUT_ALL;
            Lc.ndot = 1;
            for (int k = 0; k < nt; ++k) {
                Lc.in[k] = B(c, tb[k]);
                Lc.coef[k] = tc[k];
            }
            Lc.out = B(c, Dn);
            TRY(c, cl_lincomb(&Lc, c.N, a->slab + S_DIR, a->ws, (void*)c.st));
        }
        // (the direction's Gram row is read together with the line-search scalars below:
        //  the line search only needs D on the device)

        // ---- exact line search (AlmCore.line_search, alm.py:135) ----
        double* D = B(c, Dn);
        {
            cl_pattern P;
            c_pattern(c, D, &P);
            cl_epilogue E;
            memset(&E, 0, sizeof(E));
            E.nz = 3;
            E.Z[0] = R;
            E.Z[1] = D;
            E.Z[2] = a->CR;
            E.ndot = 3;
            E.da[0] = CL_OUT;
            E.db[0] = 16;
            E.da[1] = CL_OUT;
            E.db[1] = 17;
            E.da[2] = 18;
            E.db[2] = 17;
            TRY(c, cl_pattern_spmm(&P, D, a->ld, 1.0, &E, a->CD, a->slab + S_LS, a->ws, (void*)c.st));
            c_release(c);
        }
        if (!c.generic) {
            TRY(c, cl_diag_constraint_eval(a->n, a->aval, a->ld, R, D, D, R, a->q1, D, D, a->q2, (void*)c.st));
        } else if (a->pair != nullptr) {
            // single-entry constraints: R and D interleaved (AlmCore.line_search's pair branch)
            TRY(c, cl_pair_pack(a->n, a->ld, R, a->pair, 0, (void*)c.st));
            TRY(c, cl_pair_pack(a->n, a->ld, D, a->pair, 1, (void*)c.st));
            TRY(c, cl_constraint_eval_pair(a->m, a->con_indptr, a->con_pi, a->con_pj, a->con_val, a->ld, a->pair,
                                           a->q1, a->q2, (void*)c.st));
        } else {
            TRY(c, cl_constraint_eval(a->m, a->con_indptr, a->con_pi, a->con_pj, a->con_val, a->ld, R, D, D, R, a->q1,
                                      D, D, a->q2, (void*)c.st));
        }
        {
            cl_lincomb_args Lc;
            memset(&Lc, 0, sizeof(Lc));
            Lc.nin = 5;
            Lc.mode = CL_DOT_PAIRS;
            const double* ins[5] = {a->lam, a->b, ax_cur, a->q1, a->q2};
            const double cf[5] = {-1.0, a->rho, -a->rho, 0.0, 0.0};
            for (int k = 0; k < 5; ++k) {
                Lc.in[k] = ins[k];
                Lc.coef[k] = cf[k];
            }
            Lc.out = a->wv;
            Lc.ndot = 5;
            const uint8_t da[5] = {4, 3, CL_OUT, 3, CL_OUT}, db[5] = {4, 4, 4, 3, 3};
            for (int k = 0; k < 5; ++k) {
                Lc.da[k] = da[k];
                Lc.db[k] = db[k];
            }
            TRY(c, cl_lincomb(&Lc, c.M, a->slab + S_MV, a->ws, (void*)c.st));
        }
        if (!fetch(c, S_MV + 5)) break;
        for (int k = 0; k < nt; ++k) hist.set(Dn, tb[k], a->host[S_DIR + k]);
        hist.set(Dn, Dn, a->host[S_DIR + nt]);
        const double cdr = a->host[S_LS], cdd = a->host[S_LS + 1], crd = a->host[S_LS + 2];
        const double q2q2 = a->host[S_MV], q1q2 = a->host[S_MV + 1], wq2 = a->host[S_MV + 2];
        const double q1q1 = a->host[S_MV + 3], wq1 = a->host[S_MV + 4];
        const double p1 = a->scale * (cdr + crd);
        const double p2 = a->scale * cdd;
        const double quart[4] = {0.5 * a->rho * q2q2, a->rho * q1q2, p2 - wq2 + 0.5 * a->rho * q1q1, p1 - wq1};
        double tau = 0.0;
        const bool zero = best_step(quart, &tau);
        if (zero || tau == 0.0) {
            pool.put(Dn);
            hit = false;
            break;
        }

        // ---- step + gradient + Gram rows (AlmCore.grad_value) ----
        const bool refresh = (it + 1) % CL_ALM_REFRESH == 0;
        int H[2 * CL_ALM_MAXMEM + 1];
        int nh = 0;
        for (int k = 0; k < hist.cnt; ++k) H[nh++] = hist.at(k).d;
        for (int k = 0; k < hist.cnt; ++k) H[nh++] = hist.at(k).y;
        H[nh++] = Dn;
        if (refresh) {
            cl_lincomb_args Lc;
            memset(&Lc, 0, sizeof(Lc));
            Lc.nin = 2;
            Lc.mode = CL_DOT_PAIRS;
            Lc.in[0] = R;
            Lc.in[1] = D;
            Lc.coef[0] = 1.0;
            Lc.coef[1] = tau;
            Lc.out = R;
            TRY(c, cl_lincomb(&Lc, c.N, nullptr, nullptr, (void*)c.st));
            constraint_values(c, R, ax_cur);
            c_times(c, R, a->CR);
        }
        double* ax_out = refresh ? ax_cur : ax_alt;
        if (!grad_value(c, R, g, nullptr, gscr, yscr, H, nh, D, a->CD, tau, refresh, ax_cur, ax_out, s)) break;
        if (!refresh) {
            double* t = ax_cur;
            ax_cur = ax_alt;
            ax_alt = t;
        }
        L = a->scale * s[0] + s[3] + 0.5 * a->rho * s[4];
        gg = s[1];
        if (!(isfinite(L) && isfinite(gg))) {
            status = 2;
            break;
        }
        const int gnew = gscr, ynew = yscr;
        for (int k = 0; k < nh; ++k) hist.set(gnew, H[k], s[7 + k]);
        for (int k = 0; k < nh; ++k) hist.set(ynew, H[k], s[7 + CL_MAXIN + k]);
        hist.set(gnew, gnew, gg);
        hist.set(ynew, ynew, s[5]);
        hist.set(gnew, ynew, s[6]);
        const double ys = tau * s[2];
        bool accepted = false;
        int ev_d = -1, ev_y = -1;
        if (ys > 0.0) {
            accepted = true;
            if (hist.cnt == hist.cap) {
                const Pair& old = hist.at(0);
                ev_d = old.d;
                ev_y = old.y;
                hist.head = (hist.head + 1) % CL_ALM_MAXMEM;
                --hist.cnt;
            }
            Pair np;
            np.d = Dn;
            np.y = ynew;
            np.sigma = tau;
            np.beta = 1.0 / ys;
            hist.p[(hist.head + hist.cnt) % CL_ALM_MAXMEM] = np;
            ++hist.cnt;
        }
        gscr = g;
        g = gnew;
        if (accepted) {
            if (ev_d >= 0) {
                yscr = ev_y;
                pool.put(ev_d);
            } else {
                yscr = pool.get();
            }
        } else {
            pool.put(Dn);
            yscr = ynew;
        }
        iterations = it + 1;
        if (nrec < a->rec_cap) {
            a->rec[4 * nrec + 0] = L;
            a->rec[4 * nrec + 1] = sqrt(s[4]) / (1.0 + a->b1);
            a->rec[4 * nrec + 2] = gnorm;
            a->rec[4 * nrec + 3] = now_s();
            ++nrec;
        }
    }
    out->iterations = iterations;
    out->n_records = nrec;
    out->ax_is_ax2 = ax_cur == a->ax2;
    out->hit_cap = hit && status == 0 && !c.rc;
    out->status = status;
    out->err_line = c.line;
    return c.rc;
}

}  // namespace

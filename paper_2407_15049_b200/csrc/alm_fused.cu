// alm_fused.cu -- the ALM inner solve (alm.py:268 alm_inner) for diagonal
// constraints as ONE cooperative kernel, for problems small enough that launch
// and round-trip latency bound an iteration.
//
// cl_alm_inner_diag (alm_native.cu) runs 5 launches and 2 host synchronizes
// per L-BFGS iteration. Here the whole inner solve is one launch: thread 0 of
// every block replays the host-side scalar algebra of alm_native.cu (the
// vector-free two-loop recursion over the Gram matrix, the quartic line search
// with best_step's tie-breaking, the curvature-pair bookkeeping) from the same
// grid-reduced values, so all blocks take identical decisions; the vector passes
// between them are separated by grid barriers. Per iteration:
//
//   direction   D = sum c_k H_k (+ its Gram row)                       1 barrier
//   line search C D (gathered), <CD,R>, <CD,D>, <CR,D>, q1, q2, w dots  1 barrier
//   update      R, CR, A(RR^T), g, y, Lagrangian pieces, Gram rows     1 barrier
//
// Row arithmetic follows the multi-launch kernels; global sums are added in
// another fixed order, so iterates agree with cl_alm_inner_diag to rounding
// (tests/test_gpu_alm_native.py). Trace times come from the device global
// timer, offset to the host clock at launch.

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <time.h>
#ifdef AFZ_PROF
#include <stdio.h>
#endif

#include "culorads.h"
#include "fused_rows.cuh"
#include "fused_state.cuh"
#include "grid_bar.cuh"

namespace {

using namespace fused;

constexpr int AT = THREADS;
constexpr int AW = AT / 32;
constexpr int AMAXB = 512;                         // blocks (ws: 2 regions x AK x AMAXB doubles)
constexpr int AMAXH = 2 * CL_ALM_MAXMEM + 1;       // history operands of the update
constexpr int AK = 7 + 2 * AMAXH;                  // values of the largest reduction
constexpr int MAXB = CL_ALM_MAXBUF;
static_assert(2 * AK * AMAXB <= CL_WS_DOUBLES, "reduction regions fit the workspace");

struct AOut {
    unsigned long long ctr;  // grid-barrier arrival counter (monotonic, grid_bar.cuh)
    int iterations, n_records, n_gnorms, hit_cap, status, ax_is_ax2, err;
    unsigned long long t0;   // global timer at the start
#ifdef AFZ_PROF
    long long cyc[6];        // block 0: direction coefs, dir pass, line search, best_step, update, bookkeeping
#endif
};
__device__ AOut a_out;
__shared__ unsigned long long s_tgt;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void a_sync(unsigned) {
    const GridBar b = {&a_out.ctr, 0, &a_out.err};
    grid_bar(b, &s_tgt);
}

// Sum of K (<= AK) per-thread values over the grid, identical in every thread.
__device__ void a_reduce(double* v, int K, double* ws, int& region) {
    __shared__ double sh[AW][AK];
    __shared__ double tot[AK];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < AK; ++k) {
        if (k < K) {
            double s = v[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) sh[wid][k] = s;
        }
    }
    __syncthreads();
    double* base = ws + (int64_t)region * AK * AMAXB;
    for (int k = threadIdx.x; k < K; k += AT) {
        double s = 0.0;
        for (int w = 0; w < AW; ++w) s += sh[w][k];
        base[k * AMAXB + blockIdx.x] = s;
    }
    a_sync(gridDim.x);
    {   // warp w adds the partials of values w, w + AW, ...: all their loads in flight at once
        constexpr int KPW = (AK + AW - 1) / AW;
        double acc[KPW];
#pragma unroll
        for (int q = 0; q < KPW; ++q) acc[q] = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) {
#pragma unroll
            for (int q = 0; q < KPW; ++q) {
                const int k = wid + q * AW;
                if (k < K) acc[q] += __ldcg(base + k * AMAXB + b);
            }
        }
#pragma unroll
        for (int q = 0; q < KPW; ++q) {
            const int k = wid + q * AW;
            if (k < K) {     // warp-uniform
                double t = acc[q];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (lane == 0) tot[k] = t;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < AK; ++k)
        if (k < K) v[k] = tot[k];
    __syncthreads();
    region ^= 1;
}

// ---- host-side scalar algebra of alm_native.cu, on the device (thread 0 of every block) ----

struct Pair {
    int d, y;
    double sigma, beta;
};

__device__ int cubic_roots(double c3, double c2, double c1, double c0, double* out) {
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

__device__ double qval(const double* a, double t) { return ((a[0] * t + a[1]) * t + a[2]) * t * t + a[3] * t; }

// alm.py:202 best_step: global minimiser of the ray quartic; returns zero_direction
__device__ bool best_step(const double* a, double* tau) {
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
        if (k == 0 || vals[k] < vmin) vmin = vals[k];
    }
    const double band = vmin + 1e-12 * (1.0 + fabs(vmin));
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

// Per-block control state, owned by thread 0 (identical in every block).
struct Ctl {
    // history (ring, oldest at head) and Gram matrix over buffer indices
    int cap, cnt, head;
    Pair p[CL_ALM_MAXMEM];
    double G[MAXB][MAXB];
    int free_[MAXB];
    int nfree;
    // current iteration
    int g, gscr, yscr, Dn;
    int nt, tb[AMAXH];
    double tc[AMAXH];
    int nh, H[AMAXH];
    double tau;
    int refresh, stop, status, hit, iterations, nrec, ngn;
    double L, gg, gnorm0, gnorm;
    int ax_alt_cur;          // 1: the current constraint values live in ax2
};

__device__ __forceinline__ void gset(Ctl& c, int i, int j, double v) {
    c.G[i][j] = v;
    c.G[j][i] = v;
}
__device__ __forceinline__ const Pair& hat(const Ctl& c, int k) { return c.p[(c.head + k) % CL_ALM_MAXMEM]; }

struct Az {
    cl_alm_inner_args a;
    int G;       // lanes per row
    int h2;
    double* rec;      // device: 4 * rec_cap
    double* gnorms;   // device: rec_cap
    unsigned long long bar_base;
};

// C X for one column unit of row i (sequential over the row's slots, as the tiled SpMM)
__device__ __forceinline__ double2 c_row(const cl_pattern& P, const double* X, int h2, int64_t s0, int64_t s1, int u) {
    double2 acc = make_double2(0.0, 0.0);
    int64_t s = s0;
    for (; s + 8 <= s1; s += 8) {
        int j[8];
        double c[8];
        double2 x[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            j[t] = __ldg(P.indices + s + t);
            c[t] = __ldg(P.cv + s + t);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) x[t] = ldcg2(X + 2 * ((int64_t)j[t] * h2 + u));
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            acc.x = fma(c[t], x[t].x, acc.x);
            acc.y = fma(c[t], x[t].y, acc.y);
        }
    }
    if (s < s1) {   // the last partial chunk, predicated: its gathers are in flight together
        int j[8];
        double c[8];
        double2 x[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const bool ok = s + t < s1;
            j[t] = ok ? __ldg(P.indices + s + t) : 0;
            c[t] = ok ? __ldg(P.cv + s + t) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) x[t] = s + t < s1 ? ldcg2(X + 2 * ((int64_t)j[t] * h2 + u)) : make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < 8; ++t)
            if (s + t < s1) {
                acc.x = fma(c[t], x[t].x, acc.x);
                acc.y = fma(c[t], x[t].y, acc.y);
            }
    }
    return acc;
}

// AlmCore.grad_value (diag_update_kernel's arithmetic) over this thread's rows. fresh: the
// constraint values and C R are recomputed here (start and refresh iterations) instead of
// being stepped. v[0..7+2nh): the reductions in the layout of the update (compact: y rows at 7+nh).
__device__ void update_pass(const Az& z, const Ctl& c, bool fresh, const double* ax_in, double* ax_out,
                            const double* D, const double* gold, double* v) {
    const cl_alm_inner_args& a = z.a;
    const int G = z.G, h2 = z.h2;
    const Lanes L = lanes(G);
    const double tau = c.tau;
    const int nh = c.nh;
    double* gn = a.bufs[c.gscr];
    double* yv = a.bufs[c.yscr];
    for (int64_t i = L.first; i < a.n; i += L.stride) {
        double axr;
        const int64_t s0 = __ldg(a.cpat.indptr + i), s1 = __ldg(a.cpat.indptr + i + 1);
        if (fresh) {
            double s = 0.0;
            for (int u = L.gl; u < h2; u += G) {
                const double2 r = ldcg2(a.R + 2 * (i * h2 + u));
                s += dot2(r, r);
            }
            axr = __ldg(a.aval + i) * gsum(L, G, s);
        } else {
            axr = __ldcg(ax_in + i);
            axr = axr + tau * __ldcg(a.q1 + i) + tau * tau * __ldcg(a.q2 + i);
        }
        const double res = axr - __ldg(a.b + i);
        const double lam = __ldg(a.lam + i);
        const double w = lam + a.rho * res;
        if (L.gl == 0) {
            ax_out[i] = axr;
            v[3] += lam * res;
            v[4] += res * res;
        }
        const double wa = w * __ldg(a.aval + i);
        for (int u = L.gl; u < h2; u += G) {
            const int64_t off = 2 * (i * h2 + u);
            double2 R = ldcg2(a.R + off), CR;
            const double2 Dv = ldcg2(D + off);
            if (fresh) {
                CR = c_row(a.cpat, a.R, h2, s0, s1, u);
                st2(a.CR + off, CR);
            } else {
                CR = ldcg2(a.CR + off);
                const double2 CD = ldcg2(a.CD + off);
                R = axpy2(tau, Dv, R);
                CR = axpy2(tau, CD, CR);
                st2(a.R + off, R);
                st2(a.CR + off, CR);
            }
            double2 g;
            g.x = 2.0 * (wa * R.x + a.scale * CR.x);
            g.y = 2.0 * (wa * R.y + a.scale * CR.y);
            const double2 go = gold != nullptr ? ldcg2(gold + off) : make_double2(0.0, 0.0);
            const double2 y = make_double2(g.x - go.x, g.y - go.y);
            st2(gn + off, g);
            st2(yv + off, y);
            v[0] += dot2(CR, R);
            v[1] += dot2(g, g);
            v[2] += dot2(y, Dv);
            v[5] += dot2(y, y);
            v[6] += dot2(g, y);
#pragma unroll
            for (int h = 0; h < AMAXH; ++h)
                if (h < nh) {
                    const double2 hv = ldcg2(a.bufs[c.H[h]] + off);
                    v[7 + h] += dot2(g, hv);
                    v[7 + nh + h] += dot2(y, hv);
                }
        }
    }
}

__global__ void __launch_bounds__(AT) alm_fused_kernel(Az z) {
    __shared__ Ctl c;
    const cl_alm_inner_args& a = z.a;
    const int G = z.G, h2 = z.h2;
    const Lanes Lr = lanes(G);
    const bool t0 = threadIdx.x == 0;
    const bool writer = t0 && blockIdx.x == 0;
    double* ws = a.ws;
    int region = 0;
    double v[AK];
    if (writer) a_out.t0 = gtimer();
    if (t0) s_tgt = z.bar_base;

    if (t0) {
        c.cap = a.memory;
        c.cnt = 0;
        c.head = 0;
        c.nfree = 0;
        for (int i = a.nbuf - 1; i >= 0; --i) c.free_[c.nfree++] = i;
        c.g = c.free_[--c.nfree];
        c.gscr = c.free_[--c.nfree];
        c.yscr = c.free_[--c.nfree];
        c.nh = 0;
        c.tau = 0.0;
        c.status = 0;
        c.hit = 1;
        c.iterations = 0;
        c.nrec = 0;
        c.ngn = 0;
        c.ax_alt_cur = 0;
    }
    __syncthreads();
    // start: A(RR^T), C R and the gradient at R (grad_value with g_old = 0, D = R, fresh)
    {
        // the start writes g into the buffer the first iteration calls g (gscr/yscr roles as in alm_native.cu)
        if (t0) {
            const int t = c.gscr;
            c.gscr = c.g;
            c.g = t;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < AK; ++k) v[k] = 0.0;
        update_pass(z, c, true, a.ax, a.ax, a.R, a.zero_g, v);   // zero_g may be NULL: g_old = 0
        a_reduce(v, 7, ws, region);
        if (t0) {
            const int t = c.gscr;     // g now holds the gradient
            c.gscr = c.g;
            c.g = t;
            c.L = a.scale * v[0] + v[3] + 0.5 * a.rho * v[4];
            c.gg = v[1];
            gset(c, c.g, c.g, c.gg);
            c.stop = !(isfinite(c.L) && isfinite(c.gg));
            if (c.stop) c.status = 1;
            c.gnorm0 = sqrt(c.gg);
        }
        __syncthreads();
        if (c.stop) {
            if (writer) {
                a_out.status = 1;
                a_out.iterations = 0;
                a_out.n_records = 0;
                a_out.n_gnorms = 0;
                a_out.hit_cap = 0;
                a_out.ax_is_ax2 = 0;
            }
            return;
        }
    }

#ifdef AFZ_PROF
    long long pc[6] = {0, 0, 0, 0, 0, 0};
    long long tk = clock64();
#define AFZ_T(k) do { if (writer) { const long long _t = clock64(); pc[k] += _t - tk; tk = _t; } } while (0)
#else
#define AFZ_T(k) do { } while (0)
#endif
    for (int it = 0; it < a.max_iter; ++it) {
        AFZ_T(5);
        __syncthreads();    // every thread has read the previous c.stop before thread 0 rewrites it
        if (t0) {
            c.gnorm = sqrt(c.gg);
            if (blockIdx.x == 0 && c.ngn < a.rec_cap) z.gnorms[c.ngn] = c.gnorm;
            c.ngn = it + 1;
            c.stop = 0;
            if (c.gnorm / (1.0 + fabs(c.L)) <= a.tol) c.stop = 1;
            else if (a.reduce_factor >= 0.0 && c.gnorm <= a.reduce_factor * c.gnorm0) c.stop = 1;
            if (c.stop) c.hit = 0;
            if (!c.stop) {
                c.Dn = c.free_[--c.nfree];
                c.nt = 1;
                c.tb[0] = c.g;
                c.tc[0] = -1.0;
            }
        }
        __syncthreads();
        if (!c.stop && threadIdx.x < 32) {
            // direction coefficients (alm.py:98 via the Gram matrix, as alm_native.cu), warp 0:
            // every Gram-row dot is a warp sum, the bookkeeping is identical in all lanes
            const int ln = threadIdx.x;
            int nt = c.nt;
            double alphas[CL_ALM_MAXMEM];
            auto dotG = [&](int x) {
                double acc = ln < nt ? c.G[x][c.tb[ln]] * c.tc[ln] : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                return acc;
            };
            auto slot = [&](int buf) {     // position of buffer buf among the operands, or -1
                const unsigned hit = __ballot_sync(0xffffffffu, ln < nt && c.tb[ln] == buf);
                return hit ? __ffs(hit) - 1 : -1;
            };
            for (int k = c.cnt - 1, q = 0; k >= 0; --k, ++q) {
                const Pair pr = hat(c, k);
                const double av = pr.beta * (pr.sigma * dotG(pr.d));
                int pos = slot(pr.y);
                __syncwarp();
                if (pos < 0) {
                    if (ln == 0) {
                        c.tb[nt] = pr.y;
                        c.tc[nt] = 0.0;
                    }
                    pos = nt++;
                }
                if (ln == 0) c.tc[pos] = c.tc[pos] - av;
                __syncwarp();
                alphas[q] = av;
            }
            for (int k = 0; k < c.cnt; ++k) {
                const Pair pr = hat(c, k);
                const double av = alphas[c.cnt - 1 - k];
                const double bb = pr.beta * dotG(pr.y);
                int pos = slot(pr.d);
                __syncwarp();
                if (pos < 0) {
                    if (ln == 0) {
                        c.tb[nt] = pr.d;
                        c.tc[nt] = 0.0;
                    }
                    pos = nt++;
                }
                if (ln == 0) c.tc[pos] = c.tc[pos] + (av - bb) * pr.sigma;
                __syncwarp();
            }
            __syncwarp();   // all lanes read c.nt above (no shuffle between when the history is empty)
            if (ln == 0) c.nt = nt;
        }
        __syncthreads();
        AFZ_T(0);
        if (c.stop) break;

        // ---- direction D = sum tc_k B[tb_k] and its Gram row ----
        const int nt = c.nt;
        double* D = a.bufs[c.Dn];
#pragma unroll
        for (int k = 0; k < AK; ++k) v[k] = 0.0;
        for (int64_t i = Lr.first; i < a.n; i += Lr.stride)
            for (int u = Lr.gl; u < h2; u += G) {
                const int64_t off = 2 * (i * h2 + u);
                double2 in[AMAXH];
                double2 o = make_double2(0.0, 0.0);
#pragma unroll
                for (int k = 0; k < AMAXH; ++k)
                    if (k < nt) {
                        in[k] = ldcg2(a.bufs[c.tb[k]] + off);
                        o = axpy2(c.tc[k], in[k], o);
                    }
                st2(D + off, o);
#pragma unroll
                for (int k = 0; k < AMAXH; ++k)
                    if (k < nt) v[k] += dot2(o, in[k]);
                v[nt] += dot2(o, o);
            }
        a_reduce(v, nt + 1, ws, region);
        AFZ_T(1);
        if (t0) {
            for (int k = 0; k < nt; ++k) gset(c, c.Dn, c.tb[k], v[k]);
            gset(c, c.Dn, c.Dn, v[nt]);
        }

        // ---- exact line search (AlmCore.line_search, alm.py:135) ----
        const double* ax_cur = c.ax_alt_cur ? a.ax2 : a.ax;
        double* ax_alt = c.ax_alt_cur ? a.ax : a.ax2;
#pragma unroll
        for (int k = 0; k < AK; ++k) v[k] = 0.0;
        for (int64_t i = Lr.first; i < a.n; i += Lr.stride) {
            const int64_t s0 = __ldg(a.cpat.indptr + i), s1 = __ldg(a.cpat.indptr + i + 1);
            double x1 = 0.0, x2 = 0.0;
            for (int u = Lr.gl; u < h2; u += G) {
                const int64_t off = 2 * (i * h2 + u);
                const double2 CD = c_row(a.cpat, D, h2, s0, s1, u);
                st2(a.CD + off, CD);
                const double2 Rv = ldcg2(a.R + off), Dv = ldcg2(D + off), CRv = ldcg2(a.CR + off);
                v[0] += dot2(CD, Rv);
                v[1] += dot2(CD, Dv);
                v[2] += dot2(CRv, Dv);
                x1 += dot2(Rv, Dv) + dot2(Dv, Rv);
                x2 += dot2(Dv, Dv);
            }
            const double av = __ldg(a.aval + i);
            const double q1 = av * gsum(Lr, G, x1);
            const double q2 = av * gsum(Lr, G, x2);
            if (Lr.gl == 0) {
                a.q1[i] = q1;
                a.q2[i] = q2;
                double o = fma(-1.0, __ldg(a.lam + i), 0.0);
                o = fma(a.rho, __ldg(a.b + i), o);
                o = fma(-a.rho, __ldcg(ax_cur + i), o);
                o = fma(0.0, q1, o);
                o = fma(0.0, q2, o);
                a.wv[i] = o;
                v[3] += q2 * q2;
                v[4] += q1 * q2;
                v[5] += o * q2;
                v[6] += q1 * q1;
                v[7] += o * q1;
            }
        }
        a_reduce(v, 8, ws, region);
        AFZ_T(2);
        if (t0) {
            const double p1 = a.scale * (v[0] + v[2]);
            const double p2 = a.scale * v[1];
            const double quart[4] = {0.5 * a.rho * v[3], a.rho * v[4], p2 - v[5] + 0.5 * a.rho * v[6], p1 - v[7]};
            double tau = 0.0;
            const bool zero = best_step(quart, &tau);
            c.tau = tau;
            c.stop = 0;
            if (zero || tau == 0.0) {
                c.free_[c.nfree++] = c.Dn;
                c.hit = 0;
                c.stop = 1;
            } else {
                c.refresh = (it + 1) % CL_ALM_REFRESH == 0;
                c.nh = 0;
                for (int k = 0; k < c.cnt; ++k) c.H[c.nh++] = hat(c, k).d;
                for (int k = 0; k < c.cnt; ++k) c.H[c.nh++] = hat(c, k).y;
                c.H[c.nh++] = c.Dn;
            }
        }
        __syncthreads();
        AFZ_T(3);
        if (c.stop) break;

        // ---- step + gradient + Gram rows (AlmCore.grad_value) ----
        const bool refresh = c.refresh != 0;
        if (refresh) {   // R += tau D explicitly; A(RR^T) and C R recomputed from it
            for (int64_t i = Lr.first; i < a.n; i += Lr.stride)
                for (int u = Lr.gl; u < h2; u += G) {
                    const int64_t off = 2 * (i * h2 + u);
                    double2 o = axpy2(1.0, ldcg2(a.R + off), make_double2(0.0, 0.0));
                    o = axpy2(c.tau, ldcg2(D + off), o);
                    st2(a.R + off, o);
                }
            a_sync(gridDim.x);   // C R gathers rows of every block
        }
        double* ax_out = refresh ? const_cast<double*>(ax_cur) : ax_alt;
#pragma unroll
        for (int k = 0; k < AK; ++k) v[k] = 0.0;
        update_pass(z, c, refresh, ax_cur, ax_out, D, a.bufs[c.g], v);
        a_reduce(v, 7 + 2 * c.nh, ws, region);
        AFZ_T(4);
        if (t0) {
            if (!refresh) c.ax_alt_cur ^= 1;
            c.L = a.scale * v[0] + v[3] + 0.5 * a.rho * v[4];
            c.gg = v[1];
            if (!(isfinite(c.L) && isfinite(c.gg))) {
                c.status = 2;
                c.stop = 1;
            } else {
                const int gnew = c.gscr, ynew = c.yscr;
                for (int k = 0; k < c.nh; ++k) gset(c, gnew, c.H[k], v[7 + k]);
                for (int k = 0; k < c.nh; ++k) gset(c, ynew, c.H[k], v[7 + c.nh + k]);
                gset(c, gnew, gnew, c.gg);
                gset(c, ynew, ynew, v[5]);
                gset(c, gnew, ynew, v[6]);
                const double ys = c.tau * v[2];
                bool accepted = false;
                int ev_d = -1, ev_y = -1;
                if (ys > 0.0) {
                    accepted = true;
                    if (c.cnt == c.cap) {
                        const Pair& old = hat(c, 0);
                        ev_d = old.d;
                        ev_y = old.y;
                        c.head = (c.head + 1) % CL_ALM_MAXMEM;
                        --c.cnt;
                    }
                    Pair np;
                    np.d = c.Dn;
                    np.y = ynew;
                    np.sigma = c.tau;
                    np.beta = 1.0 / ys;
                    c.p[(c.head + c.cnt) % CL_ALM_MAXMEM] = np;
                    ++c.cnt;
                }
                c.gscr = c.g;
                c.g = gnew;
                if (accepted) {
                    if (ev_d >= 0) {
                        c.yscr = ev_y;
                        c.free_[c.nfree++] = ev_d;
                    } else {
                        c.yscr = c.free_[--c.nfree];
                    }
                } else {
                    c.free_[c.nfree++] = c.Dn;
                    c.yscr = ynew;
                }
                c.iterations = it + 1;
                if (c.nrec < a.rec_cap) {
                    if (blockIdx.x == 0) {
                        z.rec[4 * c.nrec + 0] = c.L;
                        z.rec[4 * c.nrec + 1] = sqrt(v[4]) / (1.0 + a.b1);
                        z.rec[4 * c.nrec + 2] = c.gnorm;
                        z.rec[4 * c.nrec + 3] = (double)gtimer();
                    }
                    ++c.nrec;
                }
            }
        }
        __syncthreads();
        if (c.stop) break;
    }
#ifdef AFZ_PROF
    if (writer)
        for (int k = 0; k < 6; ++k) a_out.cyc[k] = pc[k];
#endif
    if (writer) {
        a_out.iterations = c.iterations;
        a_out.n_records = c.nrec;
        a_out.n_gnorms = c.ngn;
        a_out.ax_is_ax2 = c.ax_alt_cur;
        a_out.hit_cap = c.hit && c.status == 0;
        a_out.status = c.status;
    }
}

FusedState g_state;

double host_now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

}  // namespace

extern "C" int cl_alm_inner_diag_fused(const cl_alm_inner_args* a, cl_alm_inner_stats* out) {
    if (a == nullptr || out == nullptr || a->n < 1 || a->ld < 2 || (a->ld & 1) || a->memory < 0 ||
        a->memory > CL_ALM_MAXMEM || a->nbuf < 2 * a->memory + 4 || a->nbuf > MAXB || a->rec_cap < 0 ||
        a->cpat.indptr == nullptr || (a->cpat.cv == nullptr && a->cpat.nnz > 0) ||
        (a->cpat.at_ptr != nullptr && (a->cpat.w1 != nullptr || a->cpat.w2 != nullptr)) || a->cpat.ghost != nullptr)
        return CL_EARG;
    memset(out, 0, sizeof(*out));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(a->stream);
    std::lock_guard<std::mutex> lock(g_state.mu);
    int dev = 0;
    FusedDevState* S = g_state.current(&dev);
    if (S == nullptr) return CL_EARG;
    if (S->max_blocks == 0) {
        int nb = 0, nsm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, alm_fused_kernel, AT, 0);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return (int)e;
        int mb = nb * nsm;
        if (mb > AMAXB) mb = AMAXB;
        if (mb < 1) return CL_EARG;
        S->max_blocks = mb;
    }
    const int64_t need = 5 * (int64_t)(a->rec_cap > 0 ? a->rec_cap : 1);
    if (need > S->scratch_cap) {   // this device's trace scratch; stream-ordered, no device-wide synchronize
        if (S->scratch) cudaFreeAsync(S->scratch, st);
        S->scratch = nullptr;
        S->scratch_cap = 0;
        const int64_t cap = need < 4096 ? 4096 : need;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&S->scratch), sizeof(double) * (size_t)cap, st);
        if (e != cudaSuccess) return (int)e;
        S->scratch_cap = cap;
    }
    Az z;
    z.a = *a;
    z.h2 = a->ld / 2;
    z.G = lanes_for(z.h2);
    z.rec = S->scratch;
    z.bar_base = S->bar_base;
    z.gnorms = S->scratch + 4 * (int64_t)(a->rec_cap > 0 ? a->rec_cap : 1);
    int64_t nb = (a->n * z.G + AT - 1) / AT;   // one row per lane group
    if (nb > S->max_blocks) nb = S->max_blocks;
    if (nb < 1) nb = 1;
    const double h0 = host_now();
    void* args[] = {&z};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)alm_fused_kernel, dim3((unsigned)nb), dim3(AT), args, 0, st);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbolAsync(a->host, a_out, sizeof(AOut), 0, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return (int)e;
    AOut o;
    memcpy(&o, a->host, sizeof(o));
    S->bar_base = o.ctr;
    if (o.err) {
        AOut zz;
        memset(&zz, 0, sizeof(zz));
        cudaMemcpyToSymbolAsync(a_out, &zz, sizeof(zz), 0, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
        S->bar_base = 0;
        return CL_EARG + 1;
    }
    const int nrec = o.n_records < a->rec_cap ? o.n_records : a->rec_cap;
    const int ngn = o.n_gnorms < a->rec_cap ? o.n_gnorms : a->rec_cap;
    if (nrec > 0) e = cudaMemcpy(a->rec, z.rec, sizeof(double) * 4 * (size_t)nrec, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && ngn > 0)
        e = cudaMemcpy(a->gnorms, z.gnorms, sizeof(double) * (size_t)ngn, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return (int)e;
    for (int k = 0; k < nrec; ++k)     // device timer -> host clock (the launch time is the common origin)
        a->rec[4 * k + 3] = h0 + 1e-9 * (a->rec[4 * k + 3] - (double)o.t0);
#ifdef AFZ_PROF
    fprintf(stderr, "alm_fused cycles/iter: coefs %.0f dir %.0f ls %.0f best %.0f upd %.0f book %.0f (iters %d)\n",
            (double)o.cyc[0] / o.iterations, (double)o.cyc[1] / o.iterations, (double)o.cyc[2] / o.iterations,
            (double)o.cyc[3] / o.iterations, (double)o.cyc[4] / o.iterations, (double)o.cyc[5] / o.iterations,
            o.iterations);
#endif
    out->iterations = o.iterations;
    out->n_records = o.n_records;
    out->n_gnorms = o.n_gnorms;
    out->hit_cap = o.hit_cap;
    out->status = o.status;
    out->ax_is_ax2 = o.ax_is_ax2;
    out->err_line = 0;
    return CL_OK;
}

// admm_fused.cu -- one whole ADMM step (admm.py:136 admm_step) for diagonal
// constraints as ONE cooperative kernel, for problems small enough that launch
// and host round-trip latency, not HBM, bound the step.
//
// cl_admm_step_diag (admm_native.cu) issues 8-11 launches and 1-4 host
// synchronizes per step; at n ~ 1e3-1e4 that is ~100-150 us of latency for a
// few microseconds of arithmetic. Here every phase of the step runs inside one
// launch, separated by grid-wide barriers, and the scalar decisions (tolerance
// schedule, cg_solve's stop / curvature / finiteness tests, admm.py:65) are
// taken on the device, redundantly and identically by every thread:
//
//   start         [A(UV^T)], [||A(UV^T)-b||^2], rel tolerance
//   U half-step   rhs + r0 = rhs - Q(U) (C V gathered); CG on the row-local operator
//   V half-step   rhs + r0 (C U_c gathered, C U_c stored); CG
//   step end      <C U_c, V_c>, A(U_c V_c^T), residual, dual ascent, lam_new . b
//
// Row arithmetic is the same as the multi-launch path (same expressions per row
// and per column unit); global sums are reduced in a different (fixed) order, so
// iterates agree with cl_admm_step_diag to rounding, not bit for bit
// (tests/test_gpu_admm_native.py). Reductions are deterministic: each block
// writes its partial, and after the barrier every block adds the partials in
// the same order.

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "culorads.h"
#include "fused_rows.cuh"
#include "fused_state.cuh"
#include "grid_bar.cuh"

namespace {

using namespace fused;

constexpr int FT = THREADS;             // threads per block
constexpr int FW = FT / 32;
constexpr int FMAXB = CL_RED_BLOCKS;    // partial slots per reduced value
constexpr int FK = 3;                   // values per reduction (max)

#ifndef FZ_ROWS
#define FZ_ROWS 1           // rows per lane group (grid size = n / (FT / G) / FZ_ROWS blocks)
#endif
#ifndef FZ_UNROLL
#define FZ_UNROLL 8         // gathers in flight per lane
#endif

struct FzOut {
    unsigned long long ctr;  // grid-barrier arrival counter (monotonic, grid_bar.cuh)
    cl_admm_step_stats st;
    int err;                 // a barrier timed out (the step's results are void)
};
__device__ FzOut g_out;
__shared__ unsigned long long s_tgt;

__device__ __forceinline__ void grid_sync(unsigned) {
    const GridBar b = {&g_out.ctr, 0, &g_out.err};
    grid_bar(b, &s_tgt);
}

struct Fz {
    cl_admm_diag_args a;
    int h2;      // double2 units per row
    int G;       // lanes per row (power of two <= 32)
    double rel;  // CG relative tolerance (host-independent: computed in the kernel)
    unsigned long long bar_base;
};

// Sum of K per-thread values over the whole grid, identical in every thread.
template <int K>
__device__ void greduce(double (&v)[K], double* ws, int& region) {
    __shared__ double sh[FW][FK];
    __shared__ double tot[FK];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sh[wid][k] = s;
    }
    __syncthreads();
    double* base = ws + (int64_t)region * FK * FMAXB;
    if (threadIdx.x < K) {
        double s = 0.0;
        for (int w = 0; w < FW; ++w) s += sh[w][threadIdx.x];
        base[threadIdx.x * FMAXB + blockIdx.x] = s;
    }
    grid_sync(gridDim.x);
    if (wid < K) {   // warp k adds the partials of value k: lane-strided, then a fixed tree
        double s = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) s += __ldcg(base + wid * FMAXB + b);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) tot[wid] = s;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = tot[k];
    __syncthreads();
    region ^= 1;
}

// <X_i, Y_i> over the row's units, reduced over the row's lanes (all lanes get it)
__device__ __forceinline__ double row_dot(const Lanes& L, int G, int h2, const double* X, const double* Y,
                                          int64_t i) {
    double s = 0.0;
    for (int u = L.gl; u < h2; u += G) s += dot2(ldcg2(X + 2 * (i * h2 + u)), ldcg2(Y + 2 * (i * h2 + u)));
    return gsum(L, G, s);
}

// Half-step start (cl_diag_admm_cg_init): rhs = -scale C Wf + rho Wf + a (rho b - lam) Wf,
// r = rhs - rho (a y Wf + x0), y = a <x0, Wf>; [cw = C Wf]; returns ||rhs||^2, ||r||^2.
__device__ void cg_init(const Fz& f, const double* x0, const double* Wf, double* r, double* cw, double* ws,
                        int& region, double& rhs2, double& r2) {
    const cl_admm_diag_args& a = f.a;
    const int G = f.G, h2 = f.h2;
    const Lanes L = lanes(G);
    const int64_t* __restrict__ ip = a.cpat.indptr;
    const int32_t* __restrict__ ix = a.cpat.indices;
    const double* __restrict__ cv = a.cpat.cv;
    const double alpha = -a.scale * a.cpat.c_coeff;
    double acc2[2] = {0.0, 0.0};
    for (int64_t i = L.first; i < a.n; i += L.stride) {
        const double pd = row_dot(L, G, h2, x0, Wf, i);
        const double av = __ldg(a.aval + i);
        const double nl = fma(-1.0, __ldg(a.lam + i), fma(a.rho, __ldg(a.b + i), 0.0));   // rho b - lam
        const double cq = a.rho * (av * (av * pd));
        const int64_t s0 = __ldg(ip + i), s1 = __ldg(ip + i + 1);
        for (int u = L.gl; u < h2; u += G) {
            double2 acc = make_double2(0.0, 0.0);
            int64_t s = s0;
            for (; s + FZ_UNROLL <= s1; s += FZ_UNROLL) {
                int j[FZ_UNROLL];
                double c[FZ_UNROLL];
                double2 x[FZ_UNROLL];
#pragma unroll
                for (int t = 0; t < FZ_UNROLL; ++t) {
                    j[t] = __ldg(ix + s + t);
                    c[t] = __ldg(cv + s + t);
                }
#pragma unroll
                for (int t = 0; t < FZ_UNROLL; ++t) x[t] = ldcg2(Wf + 2 * ((int64_t)j[t] * h2 + u));
#pragma unroll
                for (int t = 0; t < FZ_UNROLL; ++t) {
                    acc.x = fma(c[t], x[t].x, acc.x);
                    acc.y = fma(c[t], x[t].y, acc.y);
                }
            }
            if (s < s1) {   // the last partial chunk, predicated: its gathers are in flight together
                int j[FZ_UNROLL];
                double c[FZ_UNROLL];
                double2 x[FZ_UNROLL];
#pragma unroll
                for (int t = 0; t < FZ_UNROLL; ++t) {
                    const bool ok = s + t < s1;
                    j[t] = ok ? __ldg(ix + s + t) : 0;
                    c[t] = ok ? __ldg(cv + s + t) : 0.0;
                }
#pragma unroll
                for (int t = 0; t < FZ_UNROLL; ++t)
                    x[t] = s + t < s1 ? ldcg2(Wf + 2 * ((int64_t)j[t] * h2 + u)) : make_double2(0.0, 0.0);
#pragma unroll
                for (int t = 0; t < FZ_UNROLL; ++t)
                    if (s + t < s1) {
                        acc.x = fma(c[t], x[t].x, acc.x);
                        acc.y = fma(c[t], x[t].y, acc.y);
                    }
            }
            const int64_t off = 2 * (i * h2 + u);
            const double2 yv = ldcg2(Wf + off), zv = ldcg2(x0 + off);
            double2 o = make_double2(alpha * acc.x, alpha * acc.y);
            o = axpy2(a.rho, yv, o);
            o = axpy2(nl * av, yv, o);
            const double2 q = make_double2(fma(cq, yv.x, a.rho * zv.x), fma(cq, yv.y, a.rho * zv.y));
            double2 rr = axpy2(1.0, o, make_double2(0.0, 0.0));
            rr = axpy2(-1.0, q, rr);
            st2(r + off, rr);
            if (cw != nullptr) st2(cw + off, acc);
            acc2[0] += dot2(o, o);
            acc2[1] += dot2(rr, rr);
        }
    }
    greduce<2>(acc2, ws, region);
    rhs2 = acc2[0];
    r2 = acc2[1];
}

// CG of admm.py:65 on the row-local operator Q(p) = rho (a y Wf + p), y = a <p, Wf>, after a
// start whose residual misses eps. Returns 0 ok, 1 non-finite / 2 non-positive curvature.
// *xx = <x, x> of the final iterate (finiteness test of admm.py:98).
__device__ int cg_loop(const Fz& f, const double* x0, double* x, const double* Wf, double* r, double eps, double qr,
                       double* ws, int& region, int* its_out, double* rnorm_out, int* last_is_x, double* pq_bad,
                       double* xx) {
    const cl_admm_diag_args& a = f.a;
    const int G = f.G, h2 = f.h2;
    const Lanes L = lanes(G);
    double* p = a.p;
    int its = 0;
    double beta = 0.0, rnorm = sqrt(qr);
    const double* xs = x0;
    *last_is_x = 0;
    *xx = 0.0;
    for (int k = 0; k < a.cg_cap; ++k) {
        // p <- r + beta p; <p, Q(p)>
        double pq[1] = {0.0};
        for (int64_t i = L.first; i < a.n; i += L.stride) {
            double sd = 0.0;      // <p_i, Wf_i>, in row_dot's order
            for (int u = L.gl; u < h2; u += G) {
                const int64_t off = 2 * (i * h2 + u);
                const double2 rv = ldcg2(r + off);
                const double2 pv = beta != 0.0 ? axpy2(beta, ldcg2(p + off), rv) : rv;
                st2(p + off, pv);
                sd += dot2(pv, ldcg2(Wf + off));
            }
            sd = gsum(L, G, sd);
            const double av = __ldg(a.aval + i);
            const double c = a.rho * (av * (av * sd));
            for (int u = L.gl; u < h2; u += G) {
                const int64_t off = 2 * (i * h2 + u);
                const double2 pv = ldcg2(p + off), wv = ldcg2(Wf + off);
                const double2 q = make_double2(fma(c, wv.x, a.rho * pv.x), fma(c, wv.y, a.rho * pv.y));
                pq[0] += dot2(pv, q);
            }
        }
        greduce<1>(pq, ws, region);
        if (!isfinite(pq[0]) || pq[0] <= 0.0) {
            *last_is_x = xs == x;
            *its_out = its;
            *rnorm_out = rnorm;
            *pq_bad = pq[0];
            return isfinite(pq[0]) ? 2 : 1;
        }
        const double alpha = qr / pq[0];
        double qn[2] = {0.0, 0.0};
        for (int64_t i = L.first; i < a.n; i += L.stride) {
            const double sd = row_dot(L, G, h2, p, Wf, i);
            const double av = __ldg(a.aval + i);
            const double c = a.rho * (av * (av * sd));
            for (int u = L.gl; u < h2; u += G) {
                const int64_t off = 2 * (i * h2 + u);
                const double2 pv = ldcg2(p + off), wv = ldcg2(Wf + off);
                const double2 q = make_double2(fma(c, wv.x, a.rho * pv.x), fma(c, wv.y, a.rho * pv.y));
                const double2 xn = axpy2(alpha, pv, ldcg2(xs + off));
                const double2 rv = axpy2(-alpha, q, ldcg2(r + off));
                st2(x + off, xn);
                st2(r + off, rv);
                qn[0] += dot2(rv, rv);
                qn[1] += dot2(xn, xn);
            }
        }
        greduce<2>(qn, ws, region);
        xs = x;
        *xx = qn[1];
        rnorm = sqrt(qn[0]);
        its = k + 1;
        if (rnorm <= eps) break;
        beta = qn[0] / qr;
        qr = qn[0];
    }
    if (its == 0) {   // cg_cap == 0: the iterate is the start
        double s[1] = {0.0};
        for (int64_t i = L.first; i < a.n; i += L.stride)
            for (int u = L.gl; u < h2; u += G) {
                const int64_t off = 2 * (i * h2 + u);
                const double2 v = ldcg2(x0 + off);
                st2(x + off, v);
                s[0] += dot2(v, v);
            }
        greduce<1>(s, ws, region);
        *xx = s[0];
    }
    *its_out = its;
    *rnorm_out = rnorm;
    return 0;
}

__device__ __forceinline__ double pymax_tiny(double v) { return (1e-300 > v) ? 1e-300 : v; }

__global__ void __launch_bounds__(FT) admm_step_fused_kernel(Fz f) {
    const cl_admm_diag_args& a = f.a;
    const int G = f.G, h2 = f.h2;
    const Lanes L = lanes(G);
    double* ws = a.ws;
    int region = 0;
    cl_admm_step_stats st;
    memset(&st, 0, sizeof(st));
    const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
    if (threadIdx.x == 0) s_tgt = f.bar_base;

    // constraint values at the step start and the primal measure
    double pn2 = a.pnorm2_known;
    {
        double s[1] = {0.0};
        for (int64_t i = L.first; i < a.n; i += L.stride) {
            double ax;
            if (!a.ax_valid) {
                ax = __ldg(a.aval + i) * row_dot(L, G, h2, a.U, a.V, i);
                if (L.gl == 0) a.ax[i] = ax;
            } else {
                ax = a.ax[i];
            }
            const double d = fma(-1.0, __ldg(a.b + i), fma(1.0, ax, 0.0));
            if (L.gl == 0) s[0] += d * d;
        }
        if (!(pn2 >= 0.0)) {
            greduce<1>(s, ws, region);
            pn2 = s[0];
        }
    }
    const double pmeas = sqrt(pn2) / (1.0 + a.binf);
    const double yv = a.primal_coeff * pmeas;
    const double mn = (yv < 1e-2) ? yv : 1e-2;
    const double rel = (mn > a.rel_floor) ? mn : a.rel_floor;

    int last_is_x = 0;
    double pqb = 0.0, rhs2 = 0.0, r2 = 0.0, xx = 0.0;

    // U half-solve (admm.py:151-157)
    cg_init(f, a.U, a.V, a.r, nullptr, ws, region, rhs2, r2);
    st.eps_u = pymax_tiny(rel * sqrt(rhs2));
    double qr = r2;
    st.res_u = sqrt(qr);
    const bool u_kept = st.res_u <= st.eps_u;
    if (!u_kept) {
        const int s = cg_loop(f, a.U, a.U_new, a.V, a.r, st.eps_u, qr, ws, region, &st.it_u, &st.res_u, &last_is_x,
                              &pqb, &xx);
        if (s) {
            st.status = s; st.bad_half = 0; st.bad_is_new = last_is_x; st.pq_bad = pqb;
            if (writer) g_out.st = st;
            return;
        }
        if (!isfinite(xx)) {
            st.status = 3; st.bad_half = 0; st.bad_is_new = 1;
            if (writer) g_out.st = st;
            return;
        }
    }
    st.u_reused = u_kept;
    const double* Uc = u_kept ? a.U : a.U_new;

    // V half-solve against the new U (admm.py:159-163); stores C U_c for the step end
    cg_init(f, a.V, Uc, a.r_v, a.cu, ws, region, rhs2, r2);
    st.eps_v = pymax_tiny(rel * sqrt(rhs2));
    qr = r2;
    st.res_v = sqrt(qr);
    const bool v_kept = st.res_v <= st.eps_v;
    double xxv = 0.0;
    if (!v_kept) {
        const int s = cg_loop(f, a.V, a.V_new, Uc, a.r_v, st.eps_v, qr, ws, region, &st.it_v, &st.res_v, &last_is_x,
                              &pqb, &xxv);
        if (s) {
            st.status = s; st.bad_half = 1; st.bad_is_new = last_is_x; st.pq_bad = pqb;
            if (writer) g_out.st = st;
            return;
        }
    }
    st.v_reused = v_kept;
    const double* Vc = v_kept ? a.V : a.V_new;

    // step end (admm.py:165-166, gap inputs of admm.py:212-217), out of place
    double e[3] = {0.0, 0.0, 0.0};
    for (int64_t i = L.first; i < a.n; i += L.stride) {
        const double pd = row_dot(L, G, h2, Uc, Vc, i);
        for (int u = L.gl; u < h2; u += G) {
            const int64_t off = 2 * (i * h2 + u);
            e[0] += dot2(ldcg2(a.cu + off), ldcg2(Vc + off));
        }
        if (L.gl == 0) {
            const double ax = __ldg(a.aval + i) * pd;
            const double bb = __ldg(a.b + i);
            const double res = ax - bb;
            const double ln = fma(a.rho, res, __ldg(a.lam + i));
            a.ax[i] = ax;
            a.lam_new[i] = ln;
            e[1] += res * res;
            e[2] += ln * bb;
        }
    }
    greduce<3>(e, ws, region);
    if (!v_kept && !isfinite(xxv)) {
        st.status = 3; st.bad_half = 1; st.bad_is_new = 1;
        if (writer) g_out.st = st;
        return;
    }
    st.objective = e[0];
    st.pnorm2 = e[1];
    st.lam_b = e[2];
    st.du2 = st.dv2 = -1.0;
    if (a.want_balance) {   // admm_run's residual balancing (admm.py:184): ||U_new - U||^2, ||V_new - V||^2
        double d[2] = {0.0, 0.0};
        for (int64_t i = L.first; i < a.n; i += L.stride)
            for (int u = L.gl; u < h2; u += G) {
                const int64_t off = 2 * (i * h2 + u);
                if (!u_kept) {
                    const double2 x = ldcg2(a.U_new + off), y = ldcg2(a.U + off);
                    const double2 df = make_double2(x.x - y.x, x.y - y.y);
                    d[0] += dot2(df, df);
                }
                if (!v_kept) {
                    const double2 x = ldcg2(a.V_new + off), y = ldcg2(a.V + off);
                    const double2 df = make_double2(x.x - y.x, x.y - y.y);
                    d[1] += dot2(df, df);
                }
            }
        greduce<2>(d, ws, region);
        st.du2 = d[0];
        st.dv2 = d[1];
    }
    st.hit_cap = (st.it_u >= a.cg_cap && st.res_u > st.eps_u) || (st.it_v >= a.cg_cap && st.res_v > st.eps_v);
    if (writer) g_out.st = st;
}

FusedState g_state;

}  // namespace

extern "C" int cl_admm_step_diag_fused(const cl_admm_diag_args* a, cl_admm_step_stats* out) {
    if (a == nullptr || out == nullptr || a->n < 1 || a->ld < 2 || (a->ld & 1) || a->cg_cap < 0 ||
        a->r_v == nullptr || a->cu == nullptr || (a->cpat.cv == nullptr && a->cpat.nnz > 0) ||
        a->cpat.indptr == nullptr || a->cpat.at_ptr != nullptr ||
        a->cpat.ghost != nullptr)
        return CL_EARG;
    static_assert(sizeof(FzOut) <= 20 * sizeof(double), "the step's output fits the 20 host doubles");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(a->stream);
    std::lock_guard<std::mutex> lock(g_state.mu);
    int dev = 0;
    FusedDevState* S = g_state.current(&dev);
    if (S == nullptr) return CL_EARG;
    if (S->max_blocks == 0) {
        int nb = 0, nsm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, admm_step_fused_kernel, FT, 0);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return (int)e;
        int mb = nb * nsm;
        if (mb > FMAXB) mb = FMAXB;
        if (mb < 1) return CL_EARG;
        S->max_blocks = mb;
    }
    Fz f;
    f.a = *a;
    f.h2 = a->ld / 2;
    f.G = lanes_for(f.h2);
    f.rel = 0.0;
    f.bar_base = S->bar_base;
    // FZ_ROWS rows per lane group: latency (gather chains) against barrier cost (blocks)
    const int64_t rows_per_block = FZ_ROWS * (int64_t)(FT / f.G);
    int64_t nb = (a->n + rows_per_block - 1) / rows_per_block;
    if (nb > S->max_blocks) nb = S->max_blocks;
    if (nb < 1) nb = 1;
    void* args[] = {&f};
    cudaError_t e =
        cudaLaunchCooperativeKernel((const void*)admm_step_fused_kernel, dim3((unsigned)nb), dim3(FT), args, 0, st);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbolAsync(a->host, g_out, sizeof(FzOut), 0, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return (int)e;
    FzOut o;
    memcpy(&o, a->host, sizeof(FzOut));
    *out = o.st;
    out->err_line = 0;
    S->bar_base = o.ctr;
    if (o.err) {   // a barrier gave up: reset its state, report the step as failed
        FzOut z;
        memset(&z, 0, sizeof(z));
        cudaMemcpyToSymbolAsync(g_out, &z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
        S->bar_base = 0;
        return CL_EARG + 1;
    }
    return CL_OK;
}

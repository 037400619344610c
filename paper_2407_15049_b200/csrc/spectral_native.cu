// spectral_native.cu -- the Lanczos loop of spectral.py:28 (_lanczos_smallest) with
// native control flow, CL_LANCZOS_BATCH steps per host round trip. The operator is a pattern whose slot values are already
// assembled (C - A*(lam) on Omega, assembled once per eigenvalue estimate); per step:
// one SpMV with its Rayleigh dot, the three-term combination, two classical
// Gram-Schmidt passes against the stored basis (as the reference's full
// reorthogonalisation applied twice), the norm, and the next basis vector. Same
// launches as the Python host loop in spectral.py, so the tridiagonal
// coefficients are bit-identical (tests/test_gpu_kernels.py).

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "culorads.h"
#include "fused_state.cuh"
#include "grid_bar.cuh"

namespace {

struct Ctx {
    const cl_lanczos_args* a;
    cudaStream_t st;
    int rc;
};

bool fetch(Ctx& c, int lo, int cnt) {
    if (c.rc) return false;
    cudaError_t e = cudaMemcpyAsync(c.a->host + lo, c.a->slab + lo, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                                    c.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.st);
    if (e != cudaSuccess) c.rc = (int)e;
    return c.rc == 0;
}

}  // namespace

extern "C" int cl_lanczos_loop(const cl_lanczos_args* a, int32_t* k_out) {
    if (a == nullptr || k_out == nullptr || a->n < 1 || a->k_max < 1 || a->ldq < a->n || a->dbeta == nullptr)
        return CL_EARG;
    Ctx c;
    c.a = a;
    c.st = reinterpret_cast<cudaStream_t>(a->stream);
    c.rc = 0;
    const int64_t n = a->n;
    const int B = CL_LANCZOS_BATCH;
    // slots: [j] = alpha (<S q, q>) and [B + j] = <r, r> of the j-th step of a batch
    int k = 0;
    bool done = false;
    while (!done && k < a->k_max) {
        const int kb = (a->k_max - k) < B ? (a->k_max - k) : B;
        for (int j = 0; j < kb && !c.rc; ++j) {
            const int it = k + j;
            double* qk = a->Q + (int64_t)it * a->ldq;
            {
                cl_pattern P = a->S;
                cl_epilogue E;
                memset(&E, 0, sizeof(E));
                E.nz = 1;
                E.Z[0] = qk;
                E.ndot = 1;
                E.da[0] = CL_OUT;
                E.db[0] = 16;
                c.rc = cl_pattern_spmm(&P, qk, 1, 1.0, &E, a->u, a->slab + j, a->ws, (void*)c.st);
            }
            // r = u - alpha q_it - beta_{it-1} q_{it-1}
            if (!c.rc)
                c.rc = cl_lanczos_update(0, n, a->slab + j, it > 0 ? a->dbeta + it - 1 : nullptr, a->u, qk,
                                         it > 0 ? a->Q + (int64_t)(it - 1) * a->ldq : nullptr, a->r, nullptr,
                                         nullptr, nullptr, (void*)c.st);
            for (int pass = 0; pass < 2; ++pass) {
                if (!c.rc) c.rc = cl_basis_project(a->Q, a->ldq, it + 1, n, a->r, a->h, a->ws, (void*)c.st);
                if (!c.rc) c.rc = cl_basis_subtract(a->Q, a->ldq, it + 1, n, a->h, a->r, (void*)c.st);
            }
            {
                cl_lincomb_args L;
                memset(&L, 0, sizeof(L));
                L.nin = 1;
                L.mode = CL_DOT_PAIRS;
                L.in[0] = a->r;
                L.coef[0] = 0.0;
                L.ndot = 1;
                if (!c.rc) c.rc = cl_lincomb(&L, n, a->slab + B + j, a->ws, (void*)c.st);
            }
            // next basis vector (discarded if the stop test below ends the loop at this step)
            if (it + 1 < a->k_max && !c.rc)
                c.rc = cl_lanczos_update(1, n, nullptr, nullptr, nullptr, nullptr, nullptr, a->r, a->slab + B + j,
                                         a->dbeta + it, a->Q + (int64_t)(it + 1) * a->ldq, (void*)c.st);
        }
        if (!fetch(c, 0, 2 * B)) break;
        for (int j = 0; j < kb; ++j) {
            a->alphas[k] = a->host[j];
            ++k;
            const double beta = sqrt(a->host[B + j]);
            // scale = max(max|alpha|, 1.0) with numpy/Python semantics (a NaN alpha makes it NaN)
            double scale = 0.0;
            bool has_nan = false;
            for (int t = 0; t < k; ++t) {
                const double v = fabs(a->alphas[t]);
                if (isnan(v)) has_nan = true;
                else if (v > scale) scale = v;
            }
            scale = has_nan ? NAN : (1.0 > scale ? 1.0 : scale);
            if (k == a->k_max || beta <= a->breakdown * scale) {
                done = true;
                break;
            }
            a->betas[k - 1] = beta;
        }
    }
    *k_out = k;
    return c.rc;
}

// ---------------------------------------------------------------------------
// The whole loop as ONE cooperative launch for small n (latency-bound there):
// the stop test runs on the device, phases are separated by grid barriers, and
// global sums are reduced deterministically (per-block partials added in a fixed
// order by every block). Coefficients agree with cl_lanczos_loop to rounding.
// ---------------------------------------------------------------------------

namespace {

constexpr int LT = 256;
constexpr int LW = LT / 32;

struct LzOut {
    unsigned long long ctr;  // grid-barrier arrival counter (monotonic, grid_bar.cuh)
    int k;
    int err;
};
__device__ LzOut lz_out;
__shared__ unsigned long long s_tgt;

__device__ __forceinline__ void lz_sync(unsigned) {
    const GridBar b = {&lz_out.ctr, 0, &lz_out.err};
    grid_bar(b, &s_tgt);
}

// grid-wide sum of one value per thread, identical in every thread
__device__ double lz_sum(double v, double* ws, int& region) {
    __shared__ double sh[LW];
    __shared__ double tot;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double* base = ws + region * CL_RED_BLOCKS;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < LW; ++w) s += sh[w];
        base[blockIdx.x] = s;
    }
    lz_sync(gridDim.x);
    if (wid == 0) {
        double s = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) s += __ldcg(base + b);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) tot = s;
    }
    __syncthreads();
    const double t = tot;
    __syncthreads();
    region ^= 1;
    return t;
}

struct Lz {
    int64_t n;
    int k_max;
    double breakdown;
    double* Q;
    int64_t ldq;
    double* u;
    double* r;
    double* h;
    const int64_t* indptr;
    const int32_t* indices;
    const double* vals;
    double* alpha;
    double* beta;
    double* ws;
    unsigned long long bar_base;
};

__global__ void __launch_bounds__(LT) lanczos_fused_kernel(Lz z) {
    extern __shared__ double hs[];
    const int64_t n = z.n;
    const int64_t i0 = (int64_t)blockIdx.x * LT + threadIdx.x, di = (int64_t)gridDim.x * LT;
    const int lane = threadIdx.x & 31;
    const int gw = (int)((blockIdx.x * LT + threadIdx.x) >> 5), nw = (int)(gridDim.x * LW);
    int region = 0;
    if (threadIdx.x == 0) s_tgt = z.bar_base;
    double amax = 0.0;
    bool anan = false;
    int k = 0;
    while (k < z.k_max) {
        const double* qk = z.Q + (int64_t)k * z.ldq;
        // u = S q_k, alpha = <S q_k, q_k>
        double part = 0.0;
        for (int64_t i = i0; i < n; i += di) {
            const int64_t s0 = __ldg(z.indptr + i), s1 = __ldg(z.indptr + i + 1);
            double acc = 0.0;
            for (int64_t s = s0; s < s1; ++s) acc = fma(__ldg(z.vals + s), __ldcg(qk + __ldg(z.indices + s)), acc);
            z.u[i] = acc;
            part += acc * __ldcg(qk + i);
        }
        const double alpha = lz_sum(part, z.ws, region);
        if (blockIdx.x == 0 && threadIdx.x == 0) z.alpha[k] = alpha;
        // r = u - alpha q_k - beta_{k-1} q_{k-1}
        const double na = -alpha;
        const double nb = k > 0 ? -__ldcg(z.beta + k - 1) : 0.0;
        const double* qm = k > 0 ? z.Q + (int64_t)(k - 1) * z.ldq : nullptr;
        for (int64_t i = i0; i < n; i += di) {
            double o = fma(1.0, z.u[i], 0.0);
            o = fma(na, __ldcg(qk + i), o);
            if (qm != nullptr) o = fma(nb, __ldcg(qm + i), o);
            z.r[i] = o;
        }
        // full reorthogonalisation against q_0..q_k, twice (spectral.py:55-56)
        for (int pass = 0; pass < 2; ++pass) {
            lz_sync(gridDim.x);
            for (int t = gw; t <= k; t += nw) {       // h_t = <q_t, r>, one warp per basis vector
                const double* qt = z.Q + (int64_t)t * z.ldq;
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int64_t i = lane;
                for (; i + 96 < n; i += 128) {
                    s0 += __ldcg(qt + i) * __ldcg(z.r + i);
                    s1 += __ldcg(qt + i + 32) * __ldcg(z.r + i + 32);
                    s2 += __ldcg(qt + i + 64) * __ldcg(z.r + i + 64);
                    s3 += __ldcg(qt + i + 96) * __ldcg(z.r + i + 96);
                }
                for (; i < n; i += 32) s0 += __ldcg(qt + i) * __ldcg(z.r + i);
                double s = (s0 + s1) + (s2 + s3);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) z.h[t] = s;
            }
            lz_sync(gridDim.x);
            for (int t = threadIdx.x; t <= k; t += LT) hs[t] = __ldcg(z.h + t);
            __syncthreads();
            for (int64_t i = i0; i < n; i += di) {
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                const double* qi = z.Q + i;
                int t = 0;
                for (; t + 3 <= k; t += 4) {
                    s0 += hs[t] * __ldcg(qi + (int64_t)t * z.ldq);
                    s1 += hs[t + 1] * __ldcg(qi + (int64_t)(t + 1) * z.ldq);
                    s2 += hs[t + 2] * __ldcg(qi + (int64_t)(t + 2) * z.ldq);
                    s3 += hs[t + 3] * __ldcg(qi + (int64_t)(t + 3) * z.ldq);
                }
                for (; t <= k; ++t) s0 += hs[t] * __ldcg(qi + (int64_t)t * z.ldq);
                z.r[i] -= (s0 + s1) + (s2 + s3);
            }
        }
        ++k;
        double rr = 0.0;
        for (int64_t i = i0; i < n; i += di) {
            const double v = z.r[i];
            rr += v * v;
        }
        const double beta = sqrt(lz_sum(rr, z.ws, region));
        // scale = max(max|alpha|, 1.0) with numpy/Python semantics (a NaN alpha makes it NaN)
        const double aa = fabs(alpha);
        if (isnan(aa)) anan = true;
        else if (aa > amax) amax = aa;
        const double scale = anan ? NAN : (1.0 > amax ? 1.0 : amax);
        if (k == z.k_max || beta <= z.breakdown * scale) break;
        if (blockIdx.x == 0 && threadIdx.x == 0) z.beta[k - 1] = beta;
        const double cf = 1.0 / beta;
        double* qn = z.Q + (int64_t)k * z.ldq;
        for (int64_t i = i0; i < n; i += di) qn[i] = fma(cf, z.r[i], 0.0);
        lz_sync(gridDim.x);       // the next SpMV gathers q_k from every block
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) lz_out.k = k;
}

FusedState lz_state;

}  // namespace

extern "C" int cl_lanczos_loop_fused(const cl_lanczos_args* a, int32_t* k_out) {
    if (a == nullptr || k_out == nullptr || a->n < 1 || a->k_max < 1 || a->ldq < a->n || a->dbeta == nullptr ||
        a->dalpha == nullptr || a->S.indptr == nullptr || (a->S.cv == nullptr && a->S.nnz > 0) ||
        (a->S.at_ptr != nullptr && (a->S.w1 != nullptr || a->S.w2 != nullptr)) || a->S.ghost != nullptr)
        return CL_EARG;
    const size_t smem = sizeof(double) * (size_t)a->k_max;
    if (smem > 32 * 1024) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(a->stream);
    std::lock_guard<std::mutex> lock(lz_state.mu);
    int dev = 0;
    FusedDevState* S = lz_state.current(&dev);
    if (S == nullptr) return CL_EARG;
    if (S->max_blocks == 0) {
        int nb = 0, nsm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, lanczos_fused_kernel, LT, 32 * 1024);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return (int)e;
        int mb = nb * nsm;
        if (mb > CL_RED_BLOCKS) mb = CL_RED_BLOCKS;
        if (mb < 1) return CL_EARG;
        S->max_blocks = mb;
    }
    Lz z;
    z.n = a->n; z.k_max = a->k_max; z.breakdown = a->breakdown; z.Q = a->Q; z.ldq = a->ldq;
    z.u = a->u; z.r = a->r; z.h = a->h;
    z.indptr = a->S.indptr; z.indices = a->S.indices; z.vals = a->S.cv;
    z.alpha = a->dalpha; z.beta = a->dbeta; z.ws = a->ws;
    z.bar_base = S->bar_base;
    // one row per thread, and at least 128 warps for the projections
    int64_t nb = (a->n + LT - 1) / LT;
    if (nb < 16) nb = 16;
    if (nb > S->max_blocks) nb = S->max_blocks;
    void* args[] = {&z};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)lanczos_fused_kernel, dim3((unsigned)nb), dim3(LT), args,
                                                smem, st);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbolAsync(a->host, lz_out, sizeof(LzOut), 0, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return (int)e;
    LzOut o;
    memcpy(&o, a->host, sizeof(o));
    S->bar_base = o.ctr;
    if (o.err) {
        LzOut zz;
        memset(&zz, 0, sizeof(zz));
        cudaMemcpyToSymbolAsync(lz_out, &zz, sizeof(zz), 0, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
        S->bar_base = 0;
        return CL_EARG + 1;
    }
    const int k = o.k;
    e = cudaMemcpy(a->alphas, a->dalpha, sizeof(double) * (size_t)k, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && k > 1)
        e = cudaMemcpy(a->betas, a->dbeta, sizeof(double) * (size_t)(k - 1), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return (int)e;
    *k_out = k;
    return CL_OK;
}

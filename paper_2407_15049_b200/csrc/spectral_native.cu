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

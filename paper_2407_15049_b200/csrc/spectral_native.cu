// spectral_native.cu -- the Lanczos loop of spectral.py:28 (_lanczos_smallest) with
// native control flow. The operator is a pattern whose slot values are already
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

bool fetch(Ctx& c, int slot) {
    if (c.rc) return false;
    cudaError_t e = cudaMemcpyAsync(c.a->host + slot, c.a->slab + slot, sizeof(double), cudaMemcpyDeviceToHost, c.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.st);
    if (e != cudaSuccess) c.rc = (int)e;
    return c.rc == 0;
}

void lincomb(Ctx& c, double* out, int nin, const double* const* in, const double* coef, int64_t N, int dot_slot,
             bool out_dot) {
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
        L.da[0] = out_dot ? CL_OUT : 0;
        L.db[0] = out_dot ? CL_OUT : 0;
    }
    c.rc = cl_lincomb(&L, N, dot_slot >= 0 ? c.a->slab + dot_slot : nullptr, c.a->ws, (void*)c.st);
}

}  // namespace

extern "C" int cl_lanczos_loop(const cl_lanczos_args* a, int32_t* k_out) {
    if (a == nullptr || k_out == nullptr || a->n < 1 || a->k_max < 1 || a->ldq < a->n) return CL_EARG;
    Ctx c;
    c.a = a;
    c.st = reinterpret_cast<cudaStream_t>(a->stream);
    c.rc = 0;
    const int64_t n = a->n;
    int k = 0;
    // slots: 0 = alpha (<S q, q>), 1 = <r, r>
    while (k < a->k_max) {
        double* qk = a->Q + (int64_t)k * a->ldq;
        {
            cl_pattern P = a->S;
            cl_epilogue E;
            memset(&E, 0, sizeof(E));
            E.nz = 1;
            E.Z[0] = qk;
            E.ndot = 1;
            E.da[0] = CL_OUT;
            E.db[0] = 16;
            if (!c.rc) c.rc = cl_pattern_spmm(&P, qk, 1, 1.0, &E, a->u, a->slab + 0, a->ws, (void*)c.st);
        }
        if (!fetch(c, 0)) break;
        const double alpha = a->host[0];
        a->alphas[k] = alpha;
        if (k > 0) {
            const double* in[3] = {a->u, qk, a->Q + (int64_t)(k - 1) * a->ldq};
            const double cf[3] = {1.0, -alpha, -a->betas[k - 1]};
            lincomb(c, a->r, 3, in, cf, n, -1, false);
        } else {
            const double* in[2] = {a->u, qk};
            const double cf[2] = {1.0, -alpha};
            lincomb(c, a->r, 2, in, cf, n, -1, false);
        }
        for (int pass = 0; pass < 2; ++pass) {
            if (!c.rc) c.rc = cl_basis_project(a->Q, a->ldq, k + 1, n, a->r, a->h, a->ws, (void*)c.st);
            if (!c.rc) c.rc = cl_basis_subtract(a->Q, a->ldq, k + 1, n, a->h, a->r, (void*)c.st);
        }
        ++k;
        {
            cl_lincomb_args L;
            memset(&L, 0, sizeof(L));
            L.nin = 1;
            L.mode = CL_DOT_PAIRS;
            L.in[0] = a->r;
            L.coef[0] = 0.0;
            L.ndot = 1;
            if (!c.rc) c.rc = cl_lincomb(&L, n, a->slab + 1, a->ws, (void*)c.st);
        }
        if (!fetch(c, 1)) break;
        const double beta = sqrt(a->host[1]);
        // scale = max(max|alpha|, 1.0) with numpy/Python semantics (a NaN alpha makes it NaN)
        double scale = 0.0;
        bool has_nan = false;
        for (int t = 0; t < k; ++t) {
            const double v = fabs(a->alphas[t]);
            if (isnan(v)) has_nan = true;
            else if (v > scale) scale = v;
        }
        scale = has_nan ? NAN : (1.0 > scale ? 1.0 : scale);
        if (k == a->k_max || beta <= a->breakdown * scale) break;
        a->betas[k - 1] = beta;
        const double* in[1] = {a->r};
        const double cf[1] = {1.0 / beta};
        lincomb(c, a->Q + (int64_t)k * a->ldq, 1, in, cf, n, -1, false);
    }
    *k_out = k;
    return c.rc;
}

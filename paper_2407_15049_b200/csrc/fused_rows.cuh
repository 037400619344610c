// fused_rows.cuh -- row helpers shared by the one-launch (cooperative) kernels
// (admm_fused.cu, alm_fused.cu): 128-bit L2 loads of data written inside the
// launch, the explicitly rounded double2 dot of the multi-launch kernels, and
// the lane-group-per-row mapping.
#pragma once

#include <stdint.h>

namespace fused {

constexpr int THREADS = 256;   // threads per block of the fused kernels

// loads of data other blocks may have written in this launch go to L2 (no stale L1 lines)
__device__ __forceinline__ double2 ldcg2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }
// same rounding as dot2 of culorads.cu: y-product fused onto the rounded x-product
__device__ __forceinline__ double dot2(double2 a, double2 b) { return fma(a.y, b.y, __dmul_rn(a.x, b.x)); }
__device__ __forceinline__ double2 axpy2(double a, double2 x, double2 y) {
    return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y));
}

// A row is owned by a group of G lanes (G a power of two <= 32); gl = lane within the group.
// Rows of this thread: first, first + stride, ...
struct Lanes {
    int gl;
    unsigned mask;
    int64_t first, stride;
};

__device__ __forceinline__ Lanes lanes(int G) {
    Lanes L;
    const int lane = threadIdx.x & 31;
    L.gl = lane % G;
    L.mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - L.gl));
    L.first = ((int64_t)blockIdx.x * THREADS + threadIdx.x) / G;
    L.stride = (int64_t)gridDim.x * THREADS / G;
    return L;
}

// sum over the row's lanes (every lane of the group gets it)
__device__ __forceinline__ double gsum(const Lanes& L, int G, double s) {
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(L.mask, s, o);
    return s;
}

// lanes per row for ld doubles (ld/2 double2 units)
__host__ __device__ __forceinline__ int lanes_for(int h2) {
    return h2 <= 1 ? 1 : h2 <= 2 ? 2 : h2 <= 4 ? 4 : h2 <= 8 ? 8 : h2 <= 16 ? 16 : 32;
}

}  // namespace fused

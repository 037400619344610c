// gather_probe.cu -- DRAM bytes fetched per randomly gathered fp64 factor row (dev probe).
//
// The tiled SpMM's dominant cost on random graphs is the gather of one n x ld factor row
// per nonzero. ncu shows ~292 B of DRAM read per 208-byte row (ld 26). This probe isolates
// the gather: G random rows of X summed per lane group, written to a tiny output, with
//   ldg<LD>   LDG.128 by ld/2 lanes of a 16-lane group (the SpMM's access), rows LD doubles apart
//   bulk      one cp.async.bulk (TMA engine, 1-D) per row into a shared-memory ring
// Run plainly for time (CUDA events) and under
//   ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum
// for bytes/row.     nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

template <int LD, int LANES = 16>
__global__ void __launch_bounds__(256) ldg_gather(const double* __restrict__ X, const int* __restrict__ idx,
                                                   int64_t G, int ncols, double* out) {
    constexpr int SH = LANES == 32 ? 5 : 4;
    const int lane = threadIdx.x & (LANES - 1);
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> SH;
    const int64_t ngrp = (gridDim.x * (int64_t)blockDim.x) >> SH;
    double2 acc = make_double2(0.0, 0.0);
    const bool act = 2 * lane < ncols;
    for (int64_t k = grp * 8; k < G; k += ngrp * 8) {
        int j[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) j[u] = (k + u < G) ? __ldg(idx + k + u) : -1;
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v[u] = make_double2(0.0, 0.0);
            if (act && j[u] >= 0) v[u] = __ldg(reinterpret_cast<const double2*>(X + (int64_t)j[u] * LD) + lane);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc.x += v[u].x;
            acc.y += v[u].y;
        }
    }
    if (acc.x == 12345.678) out[0] = acc.y;   // keep the loads
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// one CTA: ring of 4 stages x 32 rows; thread 0 issues 32 bulk copies per stage
constexpr int BR = 32, NS = 4, RB = 208;
__global__ void __launch_bounds__(128) bulk_gather(const double* __restrict__ X, const int* __restrict__ idx, int64_t G,
                                                   double* out) {
    __shared__ __align__(128) double buf[NS][BR * RB / 8];
    __shared__ __align__(8) uint64_t bar[NS];
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t nch = (G + BR - 1) / BR;
    auto issue = [&](int s, int64_t ch) {
        const int64_t k0 = ch * BR;
        const int cnt = (int)min((int64_t)BR, G - k0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                     "r"((uint32_t)(cnt * RB)) : "memory");
        for (int u = 0; u < cnt; ++u) {
            const double* src = X + (int64_t)__ldg(idx + k0 + u) * (RB / 8);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(&buf[s][u * RB / 8])),
                "l"(src), "r"((uint32_t)RB), "r"(smem_u32(&bar[s]))
                : "memory");
        }
    };
    int64_t ch = blockIdx.x;
    const int64_t st = gridDim.x;
    if (tid == 0)
        for (int s = 0; s < NS && ch + s * st < nch; ++s) issue(s, ch + s * st);
    double acc = 0.0;
    uint32_t ph = 0;
    for (int it = 0; ch < nch; ch += st, ++it) {
        const int s = it % NS;
        const uint32_t par = (ph >> s) & 1u;
        asm volatile(
            "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                smem_u32(&bar[s])),
            "r"(par)
            : "memory");
        ph ^= 1u << s;
        for (int e = tid; e < BR * RB / 8; e += blockDim.x) acc += buf[s][e];
        __syncthreads();
        if (tid == 0 && ch + NS * st < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(s, ch + NS * st);
        }
    }
    if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 10000000;
    const int64_t G = argc > 2 ? atoll(argv[2]) : 60000000;
    double* X;
    int* idx;
    double* out;
    CK(cudaMalloc(&X, sizeof(double) * n * 52 + 4096));
    CK(cudaMalloc(&idx, sizeof(int) * G));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(X, 0x3F, sizeof(double) * n * 52));   // non-zero data (no compression shortcuts)
    int* h = (int*)malloc(sizeof(int) * G);
    uint64_t s = 88172645463325252ull;
    for (int64_t k = 0; k < G; ++k) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        h[k] = (int)(s % (uint64_t)n);
    }
    CK(cudaMemcpy(idx, h, sizeof(int) * G, cudaMemcpyHostToDevice));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto run = [&](const char* name, int64_t row_bytes, auto launch) {
        for (int w = 0; w < 2; ++w) launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        const int reps = 5;
        for (int r = 0; r < reps; ++r) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ms /= reps;
        const double useful = (double)G * row_bytes;
        printf("%-12s %8.3f ms  useful %.2f GB  %.0f GB/s useful  (+idx %.2f GB)\n", name, ms, useful / 1e9,
               useful / (ms * 1e6), G * 4.0 / 1e9);
    };
    const int grid = nsm * 8;
    run("ldg26", 208, [&] { ldg_gather<26><<<grid, 256>>>(X, idx, G, 26, out); });
    run("ldg28", 224, [&] { ldg_gather<28><<<grid, 256>>>(X, idx, G, 28, out); });
    run("ldg32_26", 208, [&] { ldg_gather<32><<<grid, 256>>>(X, idx, G, 26, out); });
    run("ldg32", 256, [&] { ldg_gather<32><<<grid, 256>>>(X, idx, G, 32, out); });
    run("ldg52", 416, [&] { ldg_gather<52, 32><<<grid, 256>>>(X, idx, G, 52, out); });
    run("2x ldg26", 416, [&] { ldg_gather<26><<<grid, 256>>>(X, idx, G, 26, out);
                               ldg_gather<26><<<grid, 256>>>(X + (int64_t)n * 26, idx, G, 26, out); });
    run("bulk26", 208, [&] { bulk_gather<<<nsm * 12, 128>>>(X, idx, G, out); });
    CK(cudaDeviceSynchronize());
    return 0;
}

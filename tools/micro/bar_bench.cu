// Microbenchmark: cost of the one-launch kernels' grid barrier (grid_bar.cuh) and of a
// barrier + deterministic grid sum, per call, at several grid sizes. Dev tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2407_15049_b200/csrc \
//        -o tools/micro/bar_bench tools/micro/bar_bench.cu && tools/micro/bar_bench
#include <cstdio>
#include <cuda_runtime.h>
#include "grid_bar.cuh"

__device__ unsigned long long ctr = 0;
__device__ int err = 0;
__shared__ unsigned long long s_tgt;

__global__ void bar_kernel(int iters, unsigned long long base, double* ws, double* out) {
    if (threadIdx.x == 0) s_tgt = base;
    const GridBar b = {&ctr, 0, &err};
    double acc = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        if (out != nullptr) {   // + a deterministic grid sum, as greduce does
            __shared__ double sh[8];
            double v = acc;
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
            __syncthreads();
            if (threadIdx.x == 0) {
                double s = 0;
                for (int w = 0; w < 8; ++w) s += sh[w];
                ws[(i & 1) * 1024 + blockIdx.x] = s;
            }
            grid_bar(b, &s_tgt);
            if (threadIdx.x < 32) {
                double s = 0;
                for (unsigned k = threadIdx.x; k < gridDim.x; k += 32) s += __ldcg(ws + (i & 1) * 1024 + k);
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (threadIdx.x == 0) sh[0] = s;
            }
            __syncthreads();
            acc += sh[0] * 1e-30;
            __syncthreads();
        } else {
            grid_bar(b, &s_tgt);
        }
    }
    if (out != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *out = acc;
}

int main() {
    double *ws, *out;
    cudaMalloc(&ws, 4096 * sizeof(double));
    cudaMalloc(&out, sizeof(double));
    unsigned long long base = 0;
    const int iters = 2000;
    for (int nb : {8, 25, 64, 148, 296}) {
        for (int mode = 0; mode < 2; ++mode) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            double* o = mode ? out : nullptr;
            int it = iters;
            void* args[] = {&it, &base, &ws, &o};
            cudaLaunchCooperativeKernel((const void*)bar_kernel, nb, 256, args, 0, 0);
            cudaDeviceSynchronize();
            base += (unsigned long long)nb * iters;
            cudaEventRecord(e0);
            void* args2[] = {&it, &base, &ws, &o};
            cudaLaunchCooperativeKernel((const void*)bar_kernel, nb, 256, args2, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            base += (unsigned long long)nb * iters;
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            int h_err = 0;
            cudaMemcpyFromSymbol(&h_err, err, sizeof(int));
            printf("blocks %4d  %-16s %.3f us per call  (err %d, %s)\n", nb, mode ? "barrier+sum" : "barrier",
                   1e3 * ms / iters, h_err, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}

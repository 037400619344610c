// grid_bar.cuh -- grid-wide barrier of the one-launch (cooperative) kernels.
//
// A monotonic 64-bit arrival counter per kernel family: every block adds 1 per
// barrier and waits until the counter reaches base + (barriers so far) * blocks.
// The host passes the counter's value at launch as `base` (read back after the
// previous launch), so the counter is never reset and a barrier costs one
// fire-and-forget reduction plus the acquire polls. A block that waits for
// about a second flags *err and proceeds: a fault cannot hang the GPU.
#pragma once

#include <stdint.h>

struct GridBar {
    unsigned long long* ctr;   // device counter
    unsigned long long base;   // its value at launch
    int* err;
};

__device__ __forceinline__ unsigned long long gb_load(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Thread 0 of each block keeps its next target in *tgt (shared); call from all threads.
__device__ __forceinline__ void grid_bar(const GridBar& b, unsigned long long* tgt) {
    __syncthreads();
    if (threadIdx.x == 0) {
        *tgt += gridDim.x;
        __threadfence();
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(b.ctr) : "memory");
        const long long t0 = clock64();
        while (gb_load(b.ctr) < *tgt) {
            if (clock64() - t0 > (1LL << 31)) {
                *b.err = 1;
                break;
            }
        }
    }
    __syncthreads();
}

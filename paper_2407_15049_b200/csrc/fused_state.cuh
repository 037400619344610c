// fused_state.cuh -- host-side state of the one-launch (cooperative) entry points, per device.
//
// Each family keeps, per CUDA device: the grid size its occupancy allows, the value its
// grid-barrier counter (a __device__ symbol, one instance per device) held after the last
// launch, and an optional device scratch buffer. The entry points hold the family's mutex
// for the whole call (launch + stream synchronize), so calls from several host threads or
// streams never interleave on one counter, and a call on another device never sees this
// device's counter base.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

struct FusedDevState {
    int max_blocks = 0;
    unsigned long long bar_base = 0;
    double* scratch = nullptr;
    int64_t scratch_cap = 0;
};

struct FusedState {
    static constexpr int kMaxDevices = 64;
    std::mutex mu;
    FusedDevState dev[kMaxDevices];

    // The calling thread's current device's slot (nullptr if the device id is out of range).
    FusedDevState* current(int* dev_out = nullptr) {
        int d = 0;
        if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) return nullptr;
        if (dev_out) *dev_out = d;
        return &dev[d];
    }
};

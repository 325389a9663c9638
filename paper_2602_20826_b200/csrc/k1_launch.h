// Host-side launchers for the K1 kernels (defined in k1_main.cu and
// k1_detail.cu so the two kernel families compile in parallel).
#pragma once

#include <cuda_runtime.h>

#include "k1_analysis.cuh"

namespace ds {

struct K1Occupancy {
    int grid_small = 0;  // persistent grid of the n <= 64 kernel (CTAs)
    int grid_big = 0;    // n <= 256 kernel
    int grid_retry = 0;  // 128-bit retry kernel
};

constexpr int kWarpsSmall = 4;  // WarpState<1,u64> per warp, 4 warps per CTA
constexpr int kWarpsBig = 1;    // WarpState<4,u64> (~50 KB) per CTA

// Query occupancy once per device and set the dynamic shared-memory limits.
cudaError_t k1_configure(int device, bool detail, K1Occupancy& occ);

// Launch the main pass(es) and the 128-bit retry pass on `s`. `a.retry` and
// `a.retry_count` must point to device scratch (count zeroed here).
cudaError_t k1_launch(const K1Args& a, const K1Occupancy& occ, bool any_big, bool detail, cudaStream_t s);

}  // namespace ds

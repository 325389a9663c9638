// Host-side launchers for the K1 kernels (defined in k1_main.cu and
// k1_detail.cu so the two kernel families compile in parallel).
#pragma once

#include <cuda_runtime.h>

#include "k1_analysis.cuh"

#include "k1_fast.cuh"
#include "k1_tri.cuh"

namespace ds {

struct K1Occupancy {
    int grid_small = 0;  // persistent grid of the n <= 64 kernel (CTAs)
    int grid_big = 0;    // n <= 256 kernel
    int grid_retry = 0;  // 128-bit retry kernel
    int grid_front = 0;  // split bounds pass (k1_front / k1_mid / k1_back_lane)
    int grid_mid = 0;
    int grid_back_lane = 0;  // k1_back_lane (one lane per DAG)
    int grid_fast = 0;       // k1_fast
};

constexpr int kWarpsSmall = 4;  // WarpState<1,u64> per warp, 4 warps per CTA
constexpr int kWarpsBig = 1;    // WarpState<4,u64> (~50 KB) per CTA
constexpr int kK1Counters = 12;  // u32 work counters at K1Args::retry_count (48 bytes)

// Scratch for the front/back split (K1Handoff), carved from one buffer.
inline size_t k1_handoff_bytes(u64 n_dags, u64 n_nodes) {
    return size_t(n_nodes) * (sizeof(K1Node) + 2 * 8 + 2) + size_t(n_dags) * 2 + 64 + 256 + size_t(n_dags) * 20 +
           size_t(n_dags / kSortWindow + 2) * 12;
}
inline K1Handoff k1_handoff_carve(void* base, u64 n_dags, u64 n_nodes) {
    K1Handoff h;
    h.node = static_cast<K1Node*>(base);
    u64* m = reinterpret_cast<u64*>(h.node + n_nodes);
    h.anc = m;
    h.divg = m + n_nodes;
    h.ro = reinterpret_cast<uint16_t*>(m + 2 * n_nodes);
    h.ndiv = h.ro + n_nodes;
    uintptr_t p = (reinterpret_cast<uintptr_t>(h.ndiv + n_dags) + 255) & ~uintptr_t(255);
    h.skey = reinterpret_cast<u64*>(p);
    h.perm = reinterpret_cast<u32*>(h.skey + n_dags);
    h.fb = h.perm + n_dags;
    h.l64 = h.fb + n_dags;
    h.wcnt = h.l64 + n_dags;
    return h;
}

// k1_big*.cu: DAGs above 256 nodes, one launcher per (W, word type, detail);
// configure = true sets the kernel's shared-memory limit instead of launching
#define DS_K1_BIG_DECL(NAME) cudaError_t NAME(const K1Args& a, int grid, cudaStream_t s, bool configure);
DS_K1_BIG_DECL(k1_big_8_u32_b)
DS_K1_BIG_DECL(k1_big_8_u64_b)
DS_K1_BIG_DECL(k1_big_8_u128_b)
DS_K1_BIG_DECL(k1_big_8_u32_d)
DS_K1_BIG_DECL(k1_big_8_u64_d)
DS_K1_BIG_DECL(k1_big_8_u128_d)
DS_K1_BIG_DECL(k1_big_16_u32_b)
DS_K1_BIG_DECL(k1_big_16_u64_b)
DS_K1_BIG_DECL(k1_big_16_u128_b)
DS_K1_BIG_DECL(k1_big_16_u32_d)
DS_K1_BIG_DECL(k1_big_16_u64_d)
DS_K1_BIG_DECL(k1_big_16_u128_d)
#undef DS_K1_BIG_DECL
constexpr size_t kBigScratchPerCta = sizeof(WarpState<16, u128>);  // HBM warp state of k1_big<16>
constexpr int kBigGrid = 148;

// Query occupancy once per device and set the dynamic shared-memory limits.
cudaError_t k1_configure(int device, bool detail, K1Occupancy& occ);

// Optional per-launch markers: an event recorded after each kernel launch
// (bench.py times the kernels one by one inside the timed region).
struct K1Marks {
    static constexpr int kMax = 10;
    cudaEvent_t ev[kMax];
    const char* name[kMax];
    int n = 0;
};

// Launch the main pass(es) and the 128-bit retry pass on `s`. `a.retry` and
// `a.retry_count` must point to device scratch (count zeroed here). max_n:
// the largest DAG of the batch (DS_MAX_NODES when unknown); above 256 nodes
// `a.big_q` [2 n_dags] and, above 512, `a.big_scratch` [kBigGrid x
// kBigScratchPerCta] must be set.
// With s_back and ev_split (bounds mode), the kernels from the walk-order sort
// on are launched on s_back after ev_split is recorded on s (and s_back waits
// for it): the caller's later work on s overlaps them.
cudaError_t k1_launch(const K1Args& a, const K1Occupancy& occ, u32 max_n, bool detail, cudaStream_t s,
                      K1Marks* marks = nullptr, cudaStream_t s_back = nullptr, cudaEvent_t ev_split = nullptr);

}  // namespace ds

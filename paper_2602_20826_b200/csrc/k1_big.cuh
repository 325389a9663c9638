// K1 for DAGs above 256 nodes (the reference's DAGs are unbounded; the
// paper's |V| sweep at P = 32 passes 256 nodes at depth ~9): the same
// warp-per-DAG phases as k1_analyse, with wider node masks —
//   W = 8  (256 < n <= 512):  the warp state (154-191 KB) in shared memory,
//                              one warp per CTA, one CTA per SM;
//   W = 16 (512 < n <= 1024): the warp state (~570-650 KB) in an HBM scratch
//                              slot per CTA (generic loads and atomics; L2
//                              holds a working set).
// Each word width is its own kernel: the 32-bit pass queues the DAGs whose
// intermediates overflow into big_q[0, n) (count retry_count[10]), the 64-bit
// pass takes those and queues its own overflows into big_q[n, 2n) (count
// retry_count[11]), the 128-bit pass is final — as the k1_analyse_retry tiers,
// with separate queues so the W <= 4 retry kernels never see these DAGs. The
// 32-bit pass finds its DAGs 32 at a time (one node_off pair per lane and a
// ballot), so a launch over a batch without such DAGs is cheap. Each
// (W, T, DETAIL) instantiation is compiled in its own translation unit
// (k1_big*.cu): W = 16 unrolls to ~80 s of ptxas per instantiation.
#pragma once

#include "k1_launch.h"

namespace ds {

template <int W, class T, bool DETAIL>
__global__ void __launch_bounds__(32) k1_big(const K1Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool kGlobal = W > 8;
    WarpState<W, T>& S =
        kGlobal ? *reinterpret_cast<WarpState<W, T>*>(a.big_scratch + size_t(blockIdx.x) * sizeof(WarpState<W, T>))
                : *reinterpret_cast<WarpState<W, T>*>(smem_raw);
    const int lane = threadIdx.x & 31;
    const u32 nbase = a.node_off[0], ebase = a.edge_off[0];
    constexpr int lo = W == 8 ? 256 : 512, hi = W == 8 ? 512 : DS_MAX_NODES;
    constexpr int tier = sizeof(T) == 4 ? 0 : sizeof(T) == 8 ? 1 : 2;
    u32* const qout = tier == 0 ? a.big_q : tier == 1 ? a.big_q + a.n_dags : nullptr;
    u32* const qoutc = tier == 0 ? a.retry_count + 10 : tier == 1 ? a.retry_count + 11 : nullptr;
    const PlatT<T> P{a.plat.M, RatT<T>{T(a.plat.tmin.n), T(a.plat.tmin.d)}, a.plat.minl};
    auto in_class = [&](u64 d) {
        const int n = int(a.node_off[d + 1] - a.node_off[d]);
        return n > lo && n <= hi;
    };
    if (tier == 0) {
        // a t_min that needs more than 32 bits starts in the 64-bit tier
        const bool narrow = ((a.plat.tmin.n | a.plat.tmin.d) >> 32) == 0;
#pragma unroll 1
        for (u64 base = u64(blockIdx.x) * 32; base < a.n_dags; base += u64(gridDim.x) * 32) {
            const u64 mine = base + lane;
            u32 m = __ballot_sync(FULL, mine < a.n_dags && in_class(mine));
#pragma unroll 1
            for (; m; m &= m - 1) {
                const u64 d = base + u64(__ffs(m) - 1);
                if (!narrow) {
                    if (lane == 0) qout[atomicAdd(qoutc, 1u)] = u32(d);
                    __syncwarp();
                    continue;
                }
                run_one<W, T, DETAIL>(S, lane, a, d, nbase, ebase, P, qout, qoutc);
            }
        }
    } else {
        const u32* qin = tier == 1 ? a.big_q : a.big_q + a.n_dags;
        const u32 count = a.retry_count[tier == 1 ? 10 : 11];
#pragma unroll 1
        for (u32 i = blockIdx.x; i < count; i += gridDim.x) {
            const u64 d = qin[i];
            if (!in_class(d)) continue;
            run_one<W, T, DETAIL>(S, lane, a, d, nbase, ebase, P, qout, qoutc);
        }
    }
}

// One host launcher per instantiation (each TU defines its own).
#define DS_K1_BIG_INSTANCE(W, T, D, NAME)                                                                   \
    cudaError_t NAME(const K1Args& a, int grid, cudaStream_t s, bool configure) {                           \
        const size_t smem = W > 8 ? 0 : sizeof(WarpState<W, T>);                                            \
        if (configure)                                                                                      \
            return cudaFuncSetAttribute(k1_big<W, T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        k1_big<W, T, D><<<grid, 32, smem, s>>>(a);                                                          \
        return cudaGetLastError();                                                                          \
    }

}  // namespace ds

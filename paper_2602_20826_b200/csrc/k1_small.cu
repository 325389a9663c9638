// K1 latency path: small host batches (the kept C++ API's single-task
// schedule() / analyze() / greedy_bound(), evaluate_corpus of a few tasks).
//
// The throughput path (k1_fast / k1_front / k1_mid / k1_wsort / k1_back_lane
// + retries over a chunked, multi-stream upload) costs ~8 launches and ~7
// copies — ~130 us for one 10-node DAG, 6x the reference's CPU. Here one
// kernel does everything for a batch of up to kSmallDags DAGs, one CTA (one
// warp) per DAG:
//   * inputs arrive in one H2D copy of the packed batch (or, DS_SMALL_COPY=0,
//     are read zero-copy from mapped pinned memory) and results are written
//     straight back into mapped pinned host memory (no D2H copy);
//   * the 32 -> 64 -> 128-bit word tiers run back to back in the same warp
//     (the overflow queue is a shared-memory slot, not a relaunch);
//   * in schedule-detail mode the warp first initialises its DAG's record
//     slices (what the throughput path's memsets do).
// So a call is: pack on the host, one copy, one launch, one stream synchronise.
#include "k1_launch.h"

namespace ds {

namespace {
template <class A, class B>
constexpr size_t cmax(A a, B b) {
    return size_t(a) > size_t(b) ? size_t(a) : size_t(b);
}
constexpr size_t kSmallSmem = cmax(cmax(sizeof(WarpState<1, u32>), sizeof(WarpState<4, u32>)),
                                   cmax(sizeof(WarpState<4, u64>), sizeof(WarpState<4, u128>)));
}  // namespace

template <bool DETAIL>
__global__ void __launch_bounds__(32) k1_small(const K1Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ u32 q[1];
    __shared__ u32 qc;
    const int lane = threadIdx.x;
    const u64 d = blockIdx.x;
    const u32 nbase = a.node_off[0], ebase = a.edge_off[0];
    const u32 n0 = a.node_off[d] - nbase;
    const int n = int(a.node_off[d + 1] - a.node_off[d]);
    if (DETAIL) {  // this DAG's record slices: node_block / node_div_group = -1, records zeroed
        for (int v = lane; v < n; v += 32) {
            a.det.node_block[n0 + v] = -1;
            a.det.node_div_group[n0 + v] = -1;
        }
        u64* e = reinterpret_cast<u64*>(a.det.entities + 2ull * n0);
        for (u64 k = lane; k < 2ull * n * sizeof(ds_entity_rec) / 8; k += 32) e[k] = 0;
        u64* g = reinterpret_cast<u64*>(a.det.groups + n0);
        for (u64 k = lane; k < u64(n) * sizeof(ds_group_rec) / 8; k += 32) g[k] = 0;
    }
    if (n > 256 && n <= DS_MAX_NODES) return;  // k1_big (launched after this kernel) takes it
    if (lane == 0) qc = 0;
    __syncwarp();
    const bool narrow = ((a.plat.tmin.n | a.plat.tmin.d) >> 32) == 0;
    if (narrow) {
        const PlatT<u32> P{a.plat.M, RatT<u32>{u32(a.plat.tmin.n), u32(a.plat.tmin.d)}, a.plat.minl};
        if (n > 64 && n <= DS_MAX_NODES)
            run_one<4, u32, DETAIL>(*reinterpret_cast<WarpState<4, u32>*>(smem_raw), lane, a, d, nbase, ebase, P, q,
                                    &qc);
        else
            run_one<1, u32, DETAIL>(*reinterpret_cast<WarpState<1, u32>*>(smem_raw), lane, a, d, nbase, ebase, P, q,
                                    &qc);
    } else if (lane == 0) {
        qc = 1;  // a t_min wider than 32 bits starts in the 64-bit tier
    }
    __syncwarp();
    if (qc) {
        __syncwarp();
        if (lane == 0) qc = 0;
        __syncwarp();
        const PlatT<u64> P{a.plat.M, RatT<u64>{u64(a.plat.tmin.n), u64(a.plat.tmin.d)}, a.plat.minl};
        run_one<4, u64, DETAIL>(*reinterpret_cast<WarpState<4, u64>*>(smem_raw), lane, a, d, nbase, ebase, P, q, &qc);
        __syncwarp();
        if (qc) {
            const PlatT<u128> P2{a.plat.M, RatT<u128>{u128(a.plat.tmin.n), u128(a.plat.tmin.d)}, a.plat.minl};
            run_one<4, u128, DETAIL>(*reinterpret_cast<WarpState<4, u128>*>(smem_raw), lane, a, d, nbase, ebase, P2,
                                     nullptr, nullptr);
        }
    }
}

cudaError_t k1_small_configure() {
    cudaError_t e = cudaFuncSetAttribute(k1_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmallSmem));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k1_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmallSmem));
}

cudaError_t k1_small_launch(const K1Args& a, bool detail, cudaStream_t s) {
    if (a.n_dags == 0) return cudaSuccess;
    if (detail) k1_small<true><<<unsigned(a.n_dags), 32, kSmallSmem, s>>>(a);
    else k1_small<false><<<unsigned(a.n_dags), 32, kSmallSmem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ds

// K1 kernel instantiations and launchers. Compiled twice: bounds mode (this
// file) and schedule-detail mode (k1_detail.cu defines K1_DETAIL_TU).
#include "k1_launch.h"

#include <cstdlib>

namespace ds {

namespace {
constexpr size_t kSmemSmall = sizeof(WarpState<1, u32>) * kWarpsSmall;
constexpr size_t kSmemBig = sizeof(WarpState<4, u32>) * kWarpsBig;
constexpr size_t kSmemR64 = sizeof(WarpState<4, u64>);
constexpr size_t kSmemR128 = sizeof(WarpState<4, u128>);
}  // namespace

template <bool DETAIL>
cudaError_t k1_configure_t(int device, K1Occupancy& occ) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k1_analyse<1, DETAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemSmall))))
        return e;
    if ((e = cudaFuncSetAttribute(k1_analyse<4, DETAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBig))))
        return e;
    if ((e = cudaFuncSetAttribute(k1_analyse_retry<DETAIL, u64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemR64))))
        return e;
    if ((e = cudaFuncSetAttribute(k1_analyse_retry<DETAIL, u128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kSmemR128))))
        return e;
    int o1 = 0, o4 = 0, orr = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k1_analyse<1, DETAIL>, 32 * kWarpsSmall, kSmemSmall)))
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o4, k1_analyse<4, DETAIL>, 32 * kWarpsBig, kSmemBig)))
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&orr, k1_analyse_retry<DETAIL, u128>, 32, kSmemR128)))
        return e;
    if (o1 < 1 || o4 < 1 || orr < 1) return cudaErrorInvalidConfiguration;
    if (!DETAIL) {
        if ((e = cudaFuncSetAttribute(k1_front<>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemSmall))))
            return e;
        if ((e = cudaFuncSetAttribute(k1_mid<>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemSmall))))
            return e;
        if ((e = cudaFuncSetAttribute(k1_back<>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemSmall))))
            return e;
        int of = 0, om = 0, ob = 0, obl = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&obl, k1_back_lane<>, 32 * kLaneWarps, 0))) return e;
        int obc = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&obc, k1_back_coop<>, 32 * kCoopWarps, 0))) return e;
        if (obc < 1) return cudaErrorInvalidConfiguration;
        occ.grid_back_coop = sms * obc;
        if (obl < 1) return cudaErrorInvalidConfiguration;
        // DS_K1_LANE_CTAS_PER_SM (tuning knob): fewer resident DAG walks keep
        // their hand-off state inside L2
        if (const char* env = getenv("DS_K1_LANE_CTAS_PER_SM")) {
            const int c = atoi(env);
            if (c >= 1 && c < obl) obl = c;
        }
        occ.grid_back_lane = sms * obl;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&of, k1_front<>, 32 * kWarpsSmall, kSmemSmall)))
            return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&om, k1_mid<>, 32 * kWarpsSmall, kSmemSmall)))
            return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ob, k1_back<>, 32 * kWarpsSmall, kSmemSmall)))
            return e;
        if (of < 1 || om < 1 || ob < 1) return cudaErrorInvalidConfiguration;
        occ.grid_front = sms * of;
        occ.grid_mid = sms * om;
        occ.grid_back = sms * ob;
    }
    // one full wave; warps stride over the DAGs. DS_K1_CTAS_PER_SM (tuning
    // knob) caps the resident CTAs per SM below the occupancy limit.
    if (const char* env = getenv("DS_K1_CTAS_PER_SM")) {
        const int c = atoi(env);
        if (c >= 1 && c < o1) o1 = c;
    }
    occ.grid_small = sms * o1;
    occ.grid_big = sms * o4;
    occ.grid_retry = sms * orr;
    return cudaSuccess;
}

template <bool DETAIL>
cudaError_t k1_launch_t(const K1Args& a, const K1Occupancy& occ, bool any_big, cudaStream_t s, K1Marks* marks) {
    if (marks) marks->n = 0;
    if (a.n_dags == 0) return cudaSuccess;
    int mark_i = 0;
    auto mark = [&](const char* name) -> cudaError_t {
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess || !marks || mark_i >= K1Marks::kMax) return err;
        marks->name[mark_i] = name;
        err = cudaEventRecord(marks->ev[mark_i++], s);
        marks->n = mark_i;
        return err;
    };
    // counters, contiguous: [retry, retry2, next DAG for the W=1 kernel / k1_front<>, k1_back]
    cudaError_t e = cudaMemsetAsync(a.retry_count, 0, kK1Counters * sizeof(u32), s);
    if (e != cudaSuccess) return e;
    const u64 need_small = (a.n_dags + kWarpsSmall - 1) / kWarpsSmall;
    auto cap = [&](int g) { return int(need_small < u64(g) ? need_small : u64(g)); };
    const bool split = !DETAIL && a.h.node != nullptr;
    if (split) {
        k1_front<><<<cap(occ.grid_front), 32 * kWarpsSmall, kSmemSmall, s>>>(a);
        if ((e = mark("k1_front")) != cudaSuccess) return e;
    } else {
        k1_analyse<1, DETAIL><<<cap(occ.grid_small), 32 * kWarpsSmall, kSmemSmall, s>>>(a);
        if ((e = mark("k1_analyse<1>")) != cudaSuccess) return e;
    }
    if (any_big) {
        const int gb = int(a.n_dags < u64(occ.grid_big) ? a.n_dags : u64(occ.grid_big));
        k1_analyse<4, DETAIL><<<gb, 32 * kWarpsBig, kSmemBig, s>>>(a);
        if ((e = mark("k1_analyse<4>")) != cudaSuccess) return e;
    }
    if (split && (a.mask & DS_M_PROPOSED)) {
        k1_mid<><<<cap(occ.grid_mid), 32 * kWarpsSmall, kSmemSmall, s>>>(a);
        if ((e = mark("k1_mid")) != cudaSuccess) return e;
        // one lane per DAG (default, 3.06 ms per 1M C5 DAGs); DS_K1_BACK=coop
        // adds warp-cooperative apportion at rendezvous points (4.25 ms: the
        // lanes wait for each other), DS_K1_BACK=warp one warp per DAG (4.40)
        static const int back_kind = [] {
            const char* env = getenv("DS_K1_BACK");
            return env && env[0] == 'w' ? 2 : (env && env[0] == 'c' ? 0 : 1);
        }();
        const bool warp_back = back_kind == 2;
        // shape-sorted walk order for the lane kernel (DS_K1_SORT=0: index order)
        static const bool sort_walks = [] {
            const char* env = getenv("DS_K1_SORT");
            return !(env && env[0] == '0');
        }();
        K1Args b = a;
        b.perm = nullptr;
        if (back_kind == 1 && sort_walks && a.h.skey) {
            size_t tb = a.h.sort_tmp_bytes;
            if ((e = cub::DeviceRadixSort::SortPairs(a.h.sort_tmp, tb, a.h.skey, a.h.skey2, a.h.sperm, a.h.sperm2,
                                                     int(a.n_dags), 0, 32, s)) != cudaSuccess)
                return e;
            if ((e = mark("k1_sort")) != cudaSuccess) return e;
            b.perm = a.h.sperm2;
        }
        if (back_kind == 0) {
            const u64 need = (a.n_dags + 32 * kCoopWarps - 1) / (32 * kCoopWarps);
            k1_back_coop<><<<int(need < u64(occ.grid_back_coop) ? need : u64(occ.grid_back_coop)), 32 * kCoopWarps, 0,
                             s>>>(a);
            if ((e = mark("k1_back_coop")) != cudaSuccess) return e;
        } else if (warp_back) {
            k1_back<><<<cap(occ.grid_back), 32 * kWarpsSmall, kSmemSmall, s>>>(a);
            if ((e = mark("k1_back")) != cudaSuccess) return e;
        } else {
            const u64 need = (a.n_dags + 32 * kLaneWarps - 1) / (32 * kLaneWarps);
            const int g = int(need < u64(occ.grid_back_lane) ? need : u64(occ.grid_back_lane));
            if (a.plat.M <= 255) k1_back_lane<false, 8><<<g, 32 * kLaneWarps, 0, s>>>(b);
            else k1_back_lane<false, 16><<<g, 32 * kLaneWarps, 0, s>>>(b);
            if ((e = mark("k1_back_lane")) != cudaSuccess) return e;
        }
    }
    // wider-word retries of the DAGs that overflowed 32 (then 64) bits; with
    // nothing queued each kernel reads the count and exits
    const int gr = int(a.n_dags < u64(occ.grid_retry) ? a.n_dags : u64(occ.grid_retry));
    k1_analyse_retry<DETAIL, u64><<<gr, 32, kSmemR64, s>>>(a);
    if ((e = mark("k1_analyse_retry<u64>")) != cudaSuccess) return e;
    k1_analyse_retry<DETAIL, u128><<<gr, 32, kSmemR128, s>>>(a);
    if ((e = mark("k1_analyse_retry<u128>")) != cudaSuccess) return e;
    return cudaSuccess;
}

#ifndef K1_DETAIL_TU
cudaError_t k1_configure_detail(int device, K1Occupancy& occ);
cudaError_t k1_launch_detail(const K1Args& a, const K1Occupancy& occ, bool any_big, cudaStream_t s, K1Marks* m);

cudaError_t k1_configure(int device, bool detail, K1Occupancy& occ) {
    return detail ? k1_configure_detail(device, occ) : k1_configure_t<false>(device, occ);
}
cudaError_t k1_launch(const K1Args& a, const K1Occupancy& occ, bool any_big, bool detail, cudaStream_t s,
                      K1Marks* marks) {
    return detail ? k1_launch_detail(a, occ, any_big, s, marks) : k1_launch_t<false>(a, occ, any_big, s, marks);
}
#else
cudaError_t k1_configure_detail(int device, K1Occupancy& occ) { return k1_configure_t<true>(device, occ); }
cudaError_t k1_launch_detail(const K1Args& a, const K1Occupancy& occ, bool any_big, cudaStream_t s, K1Marks* m) {
    return k1_launch_t<true>(a, occ, any_big, s, m);
}
#endif

}  // namespace ds

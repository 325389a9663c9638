// K1 kernel instantiations and launchers. Compiled twice: bounds mode (this
// file) and schedule-detail mode (k1_detail.cu defines K1_DETAIL_TU).
#include "k1_launch.h"

#include <algorithm>
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
    {
        using L = cudaError_t (*)(const K1Args&, int, cudaStream_t, bool);
        const L cfg[6] = {DETAIL ? k1_big_8_u32_d : k1_big_8_u32_b, DETAIL ? k1_big_8_u64_d : k1_big_8_u64_b,
                          DETAIL ? k1_big_8_u128_d : k1_big_8_u128_b, DETAIL ? k1_big_16_u32_d : k1_big_16_u32_b,
                          DETAIL ? k1_big_16_u64_d : k1_big_16_u64_b, DETAIL ? k1_big_16_u128_d : k1_big_16_u128_b};
        for (L f : cfg)
            if ((e = f(K1Args{}, 0, nullptr, true)) != cudaSuccess) return e;
    }
    if (!DETAIL) {
        if ((e = cudaFuncSetAttribute(k1_front<>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemSmall))))
            return e;
        if ((e = cudaFuncSetAttribute(k1_mid<>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemSmall))))
            return e;
        int of = 0, om = 0, obl = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&obl, k1_back_lane<>, 32 * kLaneWarps, 0))) return e;
        if (obl < 1) return cudaErrorInvalidConfiguration;
        // DS_K1_LANE_CTAS_PER_SM (tuning knob): fewer resident DAG walks keep
        // their hand-off state inside L2
        if (const char* env = getenv("DS_K1_LANE_CTAS_PER_SM")) {
            const int c = atoi(env);
            if (c >= 1 && c < obl) obl = c;
        }
        occ.grid_back_lane = sms * obl;
        int ofa = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ofa, k1_fast<32>, 32 * kFastWarps, 0))) return e;
        if (ofa < 1) return cudaErrorInvalidConfiguration;
        occ.grid_fast = sms * ofa;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&of, k1_front<>, 32 * kWarpsSmall, kSmemSmall)))
            return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&om, k1_mid<>, 32 * kWarpsSmall, kSmemSmall)))
            return e;
        if (of < 1 || om < 1) return cudaErrorInvalidConfiguration;
        occ.grid_front = sms * of;
        occ.grid_mid = sms * om;
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
cudaError_t k1_launch_t(const K1Args& a, const K1Occupancy& occ, u32 max_n, cudaStream_t s, K1Marks* marks,
                        cudaStream_t s_back, cudaEvent_t ev_split) {
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
    // the fused integer fast path (k1_fast.cuh) when the batch can use it:
    // t_min = 1, integer loads, M <= 1023 (DS_K1_FAST=0 disables it)
    static const bool fast_on = [] {
        const char* env = getenv("DS_K1_FAST");
        return !(env && env[0] == '0');
    }();
    const bool fast = split && fast_on && a.load_den == nullptr && a.plat.tmin.n == 1 && a.plat.tmin.d == 1 &&
                      a.plat.M <= 1023;
    // walk-key layout (walk_key in k1_analysis.cuh); DS_WALK_KEY overrides
    static const int key_mode = [] {
        const char* env = getenv("DS_WALK_KEY");
        return env ? atoi(env) : kDefaultWalkKey;
    }();
    K1Args af = a;
    af.fb_only = fast ? 1 : 0;
    af.key_mode = key_mode;
    // triangular wire form: the fast path reads it as is and only the DAGs
    // the general kernels take are widened (k1_tri.cuh); without the fast
    // path every DAG is widened first
    const bool tri = a.tri.adj != nullptr;
    const int gw = int(std::min<u64>((a.n_dags + 7) / 8, 148 * 8));  // 8 warps (DAGs) per CTA
    if (tri && !fast) {
        k_widen_tri<><<<gw, 256, 0, s>>>(a.tri, a.node_off, a.n_dags);
        if ((e = mark("k_widen_tri")) != cudaSuccess) return e;
    }
    if (fast) {
        const u64 need = (a.n_dags + kFastWarps - 1) / kFastWarps;
        const int gf = int(need < u64(occ.grid_fast) ? need : u64(occ.grid_fast));
        k1_fast<32><<<gf, 32 * kFastWarps, 0, s>>>(af);
        if ((e = mark("k1_fast<32>")) != cudaSuccess) return e;
        k1_fast<64><<<gf, 32 * kFastWarps, 0, s>>>(af);
        if ((e = mark("k1_fast<64>")) != cudaSuccess) return e;
    }
    if (split) {
        if (tri && fast) {  // the DAGs k1_fast queued for the general kernels
            k_widen_tri_list<><<<148, 256, 0, s>>>(a.tri, a.node_off, a.n_dags, a.h.fb, a.retry_count + kFbCounter);
            if ((e = mark("k_widen_tri_list")) != cudaSuccess) return e;
        }
        // every DAG, or (fast path) only those k1_fast queued
        k1_front<><<<cap(occ.grid_front), 32 * kWarpsSmall, kSmemSmall, s>>>(af);
        if ((e = mark("k1_front")) != cudaSuccess) return e;
    } else {
        k1_analyse<1, DETAIL><<<cap(occ.grid_small), 32 * kWarpsSmall, kSmemSmall, s>>>(a);
        if ((e = mark("k1_analyse<1>")) != cudaSuccess) return e;
    }
    if (max_n > 64) {
        const int gb = int(a.n_dags < u64(occ.grid_big) ? a.n_dags : u64(occ.grid_big));
        k1_analyse<4, DETAIL><<<gb, 32 * kWarpsBig, kSmemBig, s>>>(a);
        if ((e = mark("k1_analyse<4>")) != cudaSuccess) return e;
    }
    if (split && (a.mask & DS_M_PROPOSED)) {
        k1_mid<><<<cap(occ.grid_mid), 32 * kWarpsSmall, kSmemSmall, s>>>(af);
        if ((e = mark("k1_mid")) != cudaSuccess) return e;
    }
    // two-stream form: the walk-order sort, the lane walks, the big-DAG and
    // retry kernels go to s_back after an event, so the caller can overlap
    // this batch's walks with the next batch's front kernels
    if (s_back && ev_split) {
        if ((e = cudaEventRecord(ev_split, s)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(s_back, ev_split, 0)) != cudaSuccess) return e;
        s = s_back;
    }
    if (split && (a.mask & DS_M_PROPOSED)) {
        // shape-sorted walk order for the lane kernel (DS_K1_SORT=0: index order)
        static const bool sort_walks = [] {
            const char* env = getenv("DS_K1_SORT");
            return !(env && env[0] == '0');
        }();
        K1Args b = a;
        b.perm = nullptr;
        // DS_K1_WIDE_FIRST=0: lane walks in window order only (tuning knob);
        // DS_K1_HEAVY_GROUPS: the division-group count from which a compact
        // DAG's walk counts as heavy (walk_key_heavy)
        static const bool wide_first = [] {
            const char* env = getenv("DS_K1_WIDE_FIRST");
            return !(env && env[0] == '0');
        }();
        b.h.wcnt = nullptr;
        if (sort_walks && a.h.skey) {
            k1_wsort<><<<int((a.n_dags + kSortWindow - 1) / kSortWindow), kWsortThreads, 0, s>>>(
                a.h.skey, a.h.perm, a.n_dags, wide_first ? a.h.wcnt : nullptr, walk_key_heavy(key_mode));
            if ((e = mark("k1_wsort")) != cudaSuccess) return e;
            b.perm = a.h.perm;
            if (wide_first) b.h.wcnt = a.h.wcnt;
        }
        {
            const u64 need = (a.n_dags + 32 * kLaneWarps - 1) / (32 * kLaneWarps);
            const int g = int(need < u64(occ.grid_back_lane) ? need : u64(occ.grid_back_lane));
            if (a.plat.M <= 255) k1_back_lane<false, 8><<<g, 32 * kLaneWarps, 0, s>>>(b);
            else k1_back_lane<false, 16><<<g, 32 * kLaneWarps, 0, s>>>(b);
            if ((e = mark("k1_back_lane")) != cudaSuccess) return e;
        }
    }
    // DAGs above 256 nodes (k1_big*.cu): 32-bit pass, then the 64- and
    // 128-bit passes over what overflowed
    if (max_n > 256) {
        if (!a.big_q || (max_n > 512 && !a.big_scratch)) return cudaErrorInvalidValue;
        const bool w16 = max_n > 512;
        using L = cudaError_t (*)(const K1Args&, int, cudaStream_t, bool);
        const L w8[3] = {DETAIL ? k1_big_8_u32_d : k1_big_8_u32_b, DETAIL ? k1_big_8_u64_d : k1_big_8_u64_b,
                         DETAIL ? k1_big_8_u128_d : k1_big_8_u128_b};
        const L w16f[3] = {DETAIL ? k1_big_16_u32_d : k1_big_16_u32_b, DETAIL ? k1_big_16_u64_d : k1_big_16_u64_b,
                           DETAIL ? k1_big_16_u128_d : k1_big_16_u128_b};
        for (int t = 0; t < 3; ++t) {
            if ((e = w8[t](a, kBigGrid, s, false)) != cudaSuccess) return e;
            if ((e = mark("k1_big<8>")) != cudaSuccess) return e;
            if (w16) {
                if ((e = w16f[t](a, kBigGrid, s, false)) != cudaSuccess) return e;
                if ((e = mark("k1_big<16>")) != cudaSuccess) return e;
            }
        }
    }
    // wider-word retries of the DAGs that overflowed 32 (then 64) bits; with
    // nothing queued each kernel reads the count and exits
    if (tri && fast) {  // lane walks the fast path fed go back to the general kernels
        k_widen_tri_list<><<<148, 256, 0, s>>>(a.tri, a.node_off, a.n_dags, a.retry, a.retry_count);
        if ((e = mark("k_widen_tri_list")) != cudaSuccess) return e;
    }
    const int gr = int(a.n_dags < u64(occ.grid_retry) ? a.n_dags : u64(occ.grid_retry));
    k1_analyse_retry<DETAIL, u64><<<gr, 32, kSmemR64, s>>>(a);
    if ((e = mark("k1_analyse_retry<u64>")) != cudaSuccess) return e;
    k1_analyse_retry<DETAIL, u128><<<gr, 32, kSmemR128, s>>>(a);
    if ((e = mark("k1_analyse_retry<u128>")) != cudaSuccess) return e;
    return cudaSuccess;
}

#ifndef K1_DETAIL_TU
cudaError_t k1_configure_detail(int device, K1Occupancy& occ);
cudaError_t k1_launch_detail(const K1Args& a, const K1Occupancy& occ, u32 max_n, cudaStream_t s, K1Marks* m);

cudaError_t k1_configure(int device, bool detail, K1Occupancy& occ) {
    return detail ? k1_configure_detail(device, occ) : k1_configure_t<false>(device, occ);
}
cudaError_t k1_launch(const K1Args& a, const K1Occupancy& occ, u32 max_n, bool detail, cudaStream_t s,
                      K1Marks* marks, cudaStream_t s_back, cudaEvent_t ev_split) {
    return detail ? k1_launch_detail(a, occ, max_n, s, marks)
                  : k1_launch_t<false>(a, occ, max_n, s, marks, s_back, ev_split);
}
#else
cudaError_t k1_configure_detail(int device, K1Occupancy& occ) { return k1_configure_t<true>(device, occ); }
cudaError_t k1_launch_detail(const K1Args& a, const K1Occupancy& occ, u32 max_n, cudaStream_t s, K1Marks* m) {
    return k1_launch_t<true>(a, occ, max_n, s, m, nullptr, nullptr);
}
#endif

}  // namespace ds

// The triangular wire form (ds_dag_batch_tri) widened on the device into the
// arrays the general K1 kernels read: u64 loads, and each DAG's edge list in
// (from, to) order in a capacity layout (32 edges per adjacency word:
// edge_off[d] = 32 x word offset, edge_cnt[d] = edges). One warp per DAG:
// predecessor bits read out of the triangle (tri_preds), 32x32 warp
// transposes to successor masks, a scan for the output positions.
//
// With the fast path on, only the DAGs the general kernels take are widened
// (k_widen_tri_list over k1_fast's fallback list, then over the retry list
// before the wider-word passes); k1_fast reads the triangle itself.
#pragma once

#include "k1_analysis.cuh"

namespace ds {

__device__ __forceinline__ void tri_widen_dag(const TriWire& t, const u32* __restrict__ node_off, u64 n_dags, u64 d,
                                              const int lane) {
    const u32 nb = node_off[0], ab = t.adj_off[0];
    const u32 n0 = node_off[d] - nb;
    const int n = int(node_off[d + 1] - node_off[d]);
    const u32 w0 = t.adj_off[d] - ab, nw = t.adj_off[d + 1] - t.adj_off[d];
    for (int v = lane; v < n; v += 32) t.ln[n0 + v] = t.ln16[n0 + v];
    if (lane == 0) {
        t.edge_off[d] = w0 * 32u;
        if (d + 1 == n_dags) t.edge_off[n_dags] = (t.adj_off[n_dags] - ab) * 32u;
    }
    const u32* w = t.adj + w0;
    const u64 pa = tri_preds(w, nw, n, lane), pb = tri_preds(w, nw, n, lane + 32);
    // successors of u = lane (sa) and u = lane + 32 (sb): transpose
    const u32 t00 = warp_transpose32(u32(pa), lane), t10 = warp_transpose32(u32(pb), lane);
    const u32 t11 = n > 32 ? warp_transpose32(u32(pb >> 32), lane) : 0u;
    const u64 sa = (u64(t10) << 32) | t00, sb = u64(t11) << 32;
    // edges in (from, to) order: u = 0..31 (slot a), then 32..63 (slot b)
    const u32 ca = __popcll(sa), cb = __popcll(sb);
    u32 ia = ca, ib = cb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 ya = __shfl_up_sync(FULL, ia, o), yb = __shfl_up_sync(FULL, ib, o);
        if (lane >= o) {
            ia += ya;
            ib += yb;
        }
    }
    const u32 tot_a = __shfl_sync(FULL, ia, 31), tot = tot_a + __shfl_sync(FULL, ib, 31);
    u32* e = t.edges + w0 * 32u;
    u32 pos = ia - ca;
    for (u64 m = sa; m; m &= m - 1) e[pos++] = (u32(lane) << 16) | u32(__ffsll(m) - 1);
    pos = tot_a + ib - cb;
    for (u64 m = sb; m; m &= m - 1) e[pos++] = (u32(lane + 32) << 16) | u32(__ffsll(m) - 1);
    if (lane == 0) t.edge_cnt[d] = tot;
}

// every DAG of the batch
template <bool UNUSED = false>
__global__ void __launch_bounds__(256) k_widen_tri(const TriWire t, const u32* __restrict__ node_off, u64 n_dags) {
    const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
    for (u64 d = u64(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n_dags; d += warps)
        tri_widen_dag(t, node_off, n_dags, d, threadIdx.x & 31);
}

// the DAGs list[0 .. *count) (a K1 queue); edge_off[0] is set so the general
// kernels' base offset reads 0
template <bool UNUSED = false>
__global__ void __launch_bounds__(256) k_widen_tri_list(const TriWire t, const u32* __restrict__ node_off,
                                                        u64 n_dags, const u32* __restrict__ list,
                                                        const u32* __restrict__ count) {
    if (blockIdx.x == 0 && threadIdx.x == 0) t.edge_off[0] = 0;
    const u32 c = *count;
    const u32 warps = gridDim.x * (blockDim.x >> 5);
    for (u32 i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < c; i += warps)
        tri_widen_dag(t, node_off, n_dags, list[i], threadIdx.x & 31);
}

}  // namespace ds

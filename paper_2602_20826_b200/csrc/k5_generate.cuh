// K5 — corpus generation on the device: the
// reference's generate() (generator.cpp:24-96) with libstdc++'s exact
// random algorithms, one thread per DAG (seed = base + i, :98-108):
//   std::mt19937_64                      (Mt64, rng.cuh)
//   uniform_int_distribution<int|size_t> Lemire downscaling, 128-bit product
//                                        (uniform_int_dist.h:252-328; both go
//                                        through the u64 common type)
//   uniform_real_distribution<double>    (b - a) * generate_canonical + a
//                                        (random.h:1909, random.tcc:3349-3381):
//                                        double(x) / 2^64, clamped below 1
// Draw order is the contract: depth; each internal layer's width; per node in
// layer order the parent, then one coin per earlier-layer node except the
// parent; loads in id order (llround to the t_min grid, clamp at t_min; the
// exact_mean rescale after). Two passes replay the same streams: pass 1
// counts nodes and edges, pass 2 writes into the scanned offsets. Edges come
// out sorted by (from, to) — DagTask::make's order — by walking per-source
// successor masks (W words of 64 bits: DAGs of up to 64·W nodes).
#pragma once

#include "../../include/dagsched_b200.h"
#include "rng.cuh"

namespace ds {

__device__ __forceinline__ double canonical(Mt64& g) {
    const double r = __dmul_rn(__ull2double_rn(g.next()), 0x1p-64);
    return r >= 1.0 ? 0x1.fffffffffffffp-1 : r;  // nextafter(1, 0)
}

struct K5Args {
    u64 count, seed;
    int dmin, dmax, width, integer_loads, exact_mean;
    double lo, hi;         // load distribution bounds, computed on the host as generator.cpp:62-63
    double tmin_f;         // double(t_min)
    double density;
    u64 tmin_n, tmin_d;    // t_min, reduced
    u64 avg_n, avg_d;      // avg_load, reduced (exact_mean)
    u32* n_nodes;          // pass 1: per-DAG counts
    u32* n_edges;
    const u64* node_off64; // pass 2: exclusive scans of the counts
    const u64* edge_off64;
    u32* node_off;         // pass 2 outputs (the packed batch)
    u32* edge_off;
    int64_t* load_num;
    int64_t* load_den;
    u32* edges;
    int* bad;              // a load outside int64 (generator's overflow)
};

struct Q128 {  // non-negative rational, reduced
    u128 n, d;
};
__device__ __forceinline__ Q128 q128_make(u128 n, u128 d) {
    const u128 g = gcdw(n, d);
    if (g > 1) {
        n = divw(n, g);
        d = divw(d, g);
    }
    return Q128{n, d};
}
__device__ __forceinline__ bool q128_lt(Q128 a, Q128 b) { return a.n * b.d < b.n * a.d; }

template <int W, bool WRITE>
__global__ void __launch_bounds__(128) k5_generate(const K5Args a) {
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= a.count) return;
    constexpr int NMAX = 64 * W;
    Mt64 g;
    g.seed(a.seed + i);
    const int depth = int(uniform_ll(g, a.dmin, a.dmax));
    unsigned short begin[NMAX], size[NMAX];
    int L = 1, next = 1;
    begin[0] = 0;
    size[0] = 1;
    for (int l = 0; l < depth - 2; ++l) {  // host checked 2 + (dmax - 2) * width <= NMAX
        const int w = int(uniform_ll(g, 2, a.width));
        begin[L] = (unsigned short)next;
        size[L++] = (unsigned short)w;
        next += w;
    }
    const int sink = next++;
    u64 succ[NMAX][W];
    for (int v = 0; v < next; ++v)
        for (int w = 0; w < W; ++w) succ[v][w] = 0;
    u32 n_e = 0;
    for (int l = 1; l < L; ++l) {
        const int pb = begin[l - 1], ps = size[l - 1];
        for (int v = begin[l]; v < begin[l] + size[l]; ++v) {
            const u64 bit = 1ull << (v & 63);
            const int parent = pb + int(uniform_ll(g, 0, ps - 1));
            succ[parent][v >> 6] |= bit;
            ++n_e;
            for (int u = 0; u < begin[l]; ++u) {  // layers 0 .. l-1 are ids 0 .. begin[l]-1
                if (u != parent && canonical(g) < a.density) {
                    succ[u][v >> 6] |= bit;
                    ++n_e;
                }
            }
        }
    }
    for (int v = 0; v < sink; ++v) {
        u64 any = 0;
        for (int w = 0; w < W; ++w) any |= succ[v][w];
        if (!any) {
            succ[v][sink >> 6] |= 1ull << (sink & 63);
            ++n_e;
        }
    }
    if (!WRITE) {
        a.n_nodes[i] = u32(next);
        a.n_edges[i] = n_e;
        return;
    }
    const u64 n0 = a.node_off64[i], e0 = a.edge_off64[i];
    a.node_off[i] = u32(n0);
    a.edge_off[i] = u32(e0);
    if (i + 1 == a.count) {
        a.node_off[a.count] = u32(n0 + u64(next));
        a.edge_off[a.count] = u32(e0 + n_e);
    }
    u32* ew = a.edges + e0;
    int k = 0;
    for (int u = 0; u < next; ++u)
        for (int w = 0; w < W; ++w)
            for (u64 x = succ[u][w]; x; x &= x - 1) ew[k++] = (u32(u) << 16) | u32(64 * w + __ffsll(x) - 1);

    // loads (generator.cpp:62-90); the rationals are kept reduced like Frac
    int64_t* ln = a.load_num + n0;
    int64_t* ld = a.load_den + n0;
    const Q128 tmin{a.tmin_n, a.tmin_d};
    const double span = __dsub_rn(a.hi, a.lo);
    Q128 sum{0, 1};
    bool bad = false;
    for (int v = 0; v < next; ++v) {
        const double x = __dadd_rn(__dmul_rn(canonical(g), span), a.lo);
        Q128 l;
        if (a.integer_loads) {
            const long long s = llround(__ddiv_rn(x, a.tmin_f));  // >= 0: lo >= 0
            l = q128_make(u128(s) * a.tmin_n, a.tmin_d);
        } else {
            l = q128_make(u128(llround(__dmul_rn(x, 1000.0))), 1000);
        }
        if (q128_lt(l, tmin)) l = tmin;
        if (a.exact_mean) sum = q128_make(sum.n * l.d + l.n * sum.d, sum.d * l.d);
        bad |= (l.n >> 63) != 0 || (l.d >> 63) != 0;
        ln[v] = int64_t(l.n);
        ld[v] = int64_t(l.d);
    }
    if (a.exact_mean) {
        const Q128 f = q128_make(u128(a.avg_n) * u128(next) * sum.d, u128(a.avg_d) * sum.n);
        for (int v = 0; v < next; ++v) {
            Q128 l = q128_make(u128(ln[v]) * f.n, u128(ld[v]) * f.d);
            if (q128_lt(l, tmin)) l = tmin;
            bad |= (l.n >> 63) != 0 || (l.d >> 63) != 0;
            ln[v] = int64_t(l.n);
            ld[v] = int64_t(l.d);
        }
    }
    if (bad) atomicExch(a.bad, 1);
}

}  // namespace ds

// K1 — batched makespan-bound analysis, one warp per DAG (sm_100a).
//
// Device twin of the reference's per-DAG pipeline inside evaluate_corpus
// (experiment.cpp:52-79 -> method_bound :27-39):
//   DagTask::make            dag.cpp:22-138        (validation, closure, W^anc)
//   build_blocks/local_paths division.cpp:10-65
//   build_groups             division.cpp:67-126
//   apportion / schedule     scheduler.cpp:35-95, 175-427
//   bounds                   analysis.cpp:11-81
// Layout: a DAG of n <= 64*W nodes lives in the warp's shared-memory slice
// (SoA per node, W-word node masks). Node-parallel work (closure rounds,
// W^anc, ranks, head / candidate tests, per-node bounds) maps node v to lane
// v % 32; the inherently sequential parts of the greedy (group loop,
// apportion shed/fill, launch loop) run warp-uniformly over masks, so they
// neither diverge nor shuffle.
//
// Code size is a first-class constraint: the kernel is latency bound and its
// first version (everything inlined, 32.5k SASS instructions) spent 86% of its
// stall samples on instruction fetch. Every phase below is an out-of-line
// function and every rational op goes through one out-of-line copy (rat.cuh).
//
// Word width T: u64 for every DAG; DAGs whose u64 pass overflowed are re-run
// with T = u128 (k1_analyse_retry) so results are exact wherever the
// reference's 128-bit Boost rationals hold them.
//
// Parity rules reproduced: join order ascending W^anc
// ties id; heads = ungrouped block members whose unique in-block predecessor
// is grouped or absent, ranked W^anc desc ties id, truncated to M, Rule 2
// existential with >=, pick max m^max ties smaller id; apportion floor +
// clamp + shed/fill tie rules; first strict max response; candidate pool over
// pending members minus the whole division group, source test before the
// pending/released tests; time-fit launch rule; split par = mc*R; one split
// per group; residual keeps origin W^anc.
#pragma once

#include "../../include/dagsched_b200.h"
#include "rat.cuh"

namespace ds {

constexpr unsigned FULL = 0xffffffffu;

// Phases are inlined into their kernel: each kernel calls each phase once, and
// inlined the compiler sees that WarpState lives in shared memory (direct
// LDS/STS addressing instead of generic loads through a pointer argument).
// The rational primitives stay out of line (rat.cuh) — they have many sites.
#define K1_PHASE __device__ __forceinline__
constexpr int kFlatPath = 1 << 16;  // p_closure flag: every lower-bound weight is t_min

template <int W, class T>
struct WarpState {
    static constexpr int N = 64 * W;
    // Phase-disjoint fields share storage (shared memory decides how many
    // warps fit on an SM): successors die with p_ends / the backward closure
    // before the division groups are formed; the original loads die with
    // p_rank, after which the same words hold the pending loads; the
    // critical-path prefix dies with p_bounds before apportion remainders.
    u64 pred[N][W], anc[N][W], desc[N][W];
    union {
        u64 succ[N][W];
        u64 divg[N][W];  // division groups, in order
    };
    union {
        T ln[N];  // original load
        T pn[N];  // pending load (residual after a split)
    };
    union {
        T ld[N];
        T pd[N];
    };
    T xn[N], xd[N];  // W^anc, later per-member exec
    union {
        T cn[N];  // critical-path prefix (lower bound)
        T rn[N];  // apportion remainder (unreduced)
    };
    union {
        T cd[N];
        T rd[N];
    };
    int mmax[N];      // max_parallelism(original load)
    int mq[N];        // apportioned parallelism
    int cap[N];       // min(max_parallelism(pending load), M)
    short rank[N];    // position in (W^anc desc, id asc)
    short order[N];   // node at rank r
    short jorder[N];  // joins in (W^anc asc, id asc)
    unsigned short gen[N];   // split generation counter
    unsigned char ppart[N];  // pending entity part (0 whole, 2 residual)
    u64 rmask[W];            // rank-space scratch
    T bn[DS_N_BOUNDS], bd[DS_N_BOUNDS];  // results
};

template <int W>
struct Mask {
    u64 w[W];
    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int k = 0; k < W; ++k) w[k] = 0;
    }
    __device__ __forceinline__ bool any() const {
        u64 a = 0;
#pragma unroll
        for (int k = 0; k < W; ++k) a |= w[k];
        return a != 0;
    }
    __device__ __forceinline__ int popc() const {
        int c = 0;
#pragma unroll
        for (int k = 0; k < W; ++k) c += __popcll(w[k]);
        return c;
    }
    __device__ __forceinline__ bool test(int i) const { return (w[i >> 6] >> (i & 63)) & 1; }
    __device__ __forceinline__ void set(int i) { w[i >> 6] |= 1ull << (i & 63); }
    __device__ __forceinline__ bool eq(const Mask& o) const {
        bool e = true;
#pragma unroll
        for (int k = 0; k < W; ++k) e &= w[k] == o.w[k];
        return e;
    }
};

template <int W>
__device__ __forceinline__ Mask<W> load_mask(const u64 (&m)[W]) {
    Mask<W> r;
#pragma unroll
    for (int k = 0; k < W; ++k) r.w[k] = m[k];
    return r;
}

// Uniform mask from a per-node predicate evaluated by the owning lanes. The
// predicate body is instantiated once per mask word.
template <int W, class Pred>
__device__ __forceinline__ Mask<W> ballot_nodes(int lane, int n, Pred pred) {
    Mask<W> r;
#pragma unroll
    for (int k = 0; k < W; ++k) {
        u64 acc = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (k * 64 + h * 32 >= n) break;  // uniform: most DAGs fit one 32-node half
            acc |= u64(__ballot_sync(FULL, pred(k * 64 + h * 32 + lane))) << (32 * h);
        }
        r.w[k] = acc;
    }
    return r;
}

// Sets bit i of a 64-bit word in shared memory with a native 32-bit atomicOr
// on the half that holds it (a 64-bit atomicOr on shared memory compiles to a
// CAS spin loop, ATOMS.CAST.SPIN.64).
__device__ __forceinline__ void smem_set_bit(u64* words, int i) {
    atomicOr(reinterpret_cast<unsigned int*>(words) + (i >> 5), 1u << (i & 31));
}

// Set bits of a uniform mask, ascending. Walks each word as two 32-bit
// halves (one body instantiation): 32-bit find-first-set and clear-lowest
// take half the instructions of their 64-bit forms, and most DAGs have their
// nodes in the low half.
template <int W, class F>
__device__ __forceinline__ void for_bits(const Mask<W>& m, F f) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
        u32 lo = u32(m.w[k]), hi = u32(m.w[k] >> 32);
        int base = k * 64;
#pragma unroll 1
        for (;;) {
            if (!lo) {
                if (!hi) break;
                lo = hi;
                hi = 0;
                base = k * 64 + 32;
            }
            const int b = base + __ffs(lo) - 1;
            lo &= lo - 1;
            f(b);
        }
    }
}

// Ascending bitonic sorts of two independent key sets of up to 64 keys each,
// held as (a: element lane, b: element lane + 32) and (c, d) likewise;
// afterwards element e of each sorted order is in lane e % 32. The network
// runs as a loop (not unrolled: the kernel is instruction-fetch bound) up to
// size K (32 when every key fits the a/c halves, else 64).
template <class K_t>
__device__ __forceinline__ void bitonic64x2(K_t& a, K_t& b, K_t& c, K_t& d, const int lane, const int K) {
#pragma unroll 1
    for (int k = 2; k <= K; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {  // partners are the two registers of one lane (k == 64: ascending)
                const K_t lo = min(a, b), hi = max(a, b), lo2 = min(c, d), hi2 = max(c, d);
                a = lo;
                b = hi;
                c = lo2;
                d = hi2;
                continue;
            }
            const K_t pa = __shfl_xor_sync(FULL, a, j), pb = __shfl_xor_sync(FULL, b, j);
            const K_t pc = __shfl_xor_sync(FULL, c, j), pd = __shfl_xor_sync(FULL, d, j);
            const bool lower = (lane & j) == 0;          // this element has the smaller index
            const bool up_a = (lane & k) == 0;           // element lane: ascending run?
            const bool up_b = ((lane + 32) & k) == 0;    // element lane + 32
            a = (lower == up_a) ? min(a, pa) : max(a, pa);
            b = (lower == up_b) ? min(b, pb) : max(b, pb);
            c = (lower == up_a) ? min(c, pc) : max(c, pc);
            d = (lower == up_b) ? min(d, pd) : max(d, pd);
        }
    }
}

template <class T>
__device__ __forceinline__ bool fits_i64(T v) {
    if constexpr (sizeof(T) <= 4) return true;
    else return (v >> 63) == 0;
}

struct DetailOut {
    ds_entity_rec* ent;  // this DAG's entity slots
    ds_group_rec* grp;   // this DAG's group slots
    short* node_block;
    short* node_div_group;
    uint64_t* unl;       // this DAG's unlaunched-candidate masks (NULL: not kept)
    int unl_w;           // words per mask: ceil(n / 64)
};

// --------------------------------------------------------------- phase: loads
// dag.cpp:35-41: load >= min_load (P.minl: t_min, 1, or only > 0). A load
// below t_min is also flagged: it fails schedule() (scheduler.cpp:177-182),
// not the other bounds. Returns status | (integer_loads << 8) | (low_t << 9).
template <int W, class T>
K1_PHASE int p_load(WarpState<W, T>& S, const int lane, const int n, const u64* __restrict__ lnum,
                                   const u64* __restrict__ lden, const PlatT<T> P) {
    bool bad_load = false, bad_arg = false, frac = false, ovf = false, low_t = false;
#pragma unroll 1
    for (int v = lane; v < n; v += 32) {
        long long a = (long long)lnum[v];
        long long b = lden ? (long long)lden[v] : 1;
        if (b == 0) bad_arg = true;
        if (b < 0) {
            a = -a;
            b = -b;
        }
        RatT<T> l{0, 1};
        const bool too_wide = sizeof(T) == 4 && a > 0 && b > 0 && ((u64(a) | u64(b)) >> 32) != 0;
        if (too_wide) {
            ovf = true;  // handled by a wider tier
            l = P.tmin;
        } else if (a > 0 && b > 0) {
            l = n_reduce<T>(T(u64(a)), T(u64(b)));
        }
        if (a <= 0) {
            bad_load = true;
        } else if (!too_wide) {
            const bool lt = n_cmp(l, P.tmin) < 0;
            low_t |= lt;
            bad_load |= P.minl == 0 ? lt : (P.minl == 1 && l.n < l.d);  // canonical: l < 1 iff n < d
        }
        frac |= l.d != 1;
        S.ln[v] = l.n;
        S.ld[v] = l.d;
        int mp = 1;
        if (a > 0 && b > 0) {
            mp = q_max_par(l, P);
            if (mp < 0) ovf = true;
        }
        S.mmax[v] = mp;
        S.gen[v] = 0;
        S.ppart[v] = 0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            S.pred[v][k] = 0;
            S.succ[v][k] = 0;
            S.anc[v][k] = 0;
            S.desc[v][k] = 0;
        }
    }
    if (__any_sync(FULL, bad_arg)) return DS_EINVAL;
    if (__any_sync(FULL, bad_load)) return DS_E_LOAD;
    if (__any_sync(FULL, ovf)) return DS_EOVERFLOW;
    return DS_OK | ((!__any_sync(FULL, frac)) << 8) | (__any_sync(FULL, low_t) << 9);
}

// --------------------------------------------------------------- phase: edges
// dag.cpp:48-67: checked in sorted (from, to) order; the first failure wins.
template <int W, class T>
K1_PHASE int p_edges(WarpState<W, T>& S, const int lane, const int n, const u32* __restrict__ edges,
                                    const int n_edges) {
    u32 first_bad = 0xffffffffu;
    int bad_kind = 0;
#pragma unroll 1
    for (int e = lane; e < n_edges; e += 32) {
        const u32 w = edges[e];
        const int u = int(w >> 16), v = int(w & 0xffffu);
        if (u >= n || v >= n || u == v) {
            if (w < first_bad) {
                first_bad = w;
                bad_kind = (u >= n || v >= n) ? DS_E_EDGE : DS_E_SELFLOOP;
            }
        } else {
            smem_set_bit(S.succ[u], v);
            smem_set_bit(S.pred[v], u);
        }
    }
    const u32 m = __reduce_min_sync(FULL, first_bad);
    __syncwarp();
    if (m == 0xffffffffu) return DS_OK;
    const u32 who = __ballot_sync(FULL, first_bad == m);
    return __shfl_sync(FULL, bad_kind, __ffs(who) - 1);
}

// ------------------------------------------------------------ phase: closure
// dag.cpp:69-124, level-synchronous Kahn. Round r makes ready every node whose
// predecessors (successors when !FWD) are all processed; round = 1 + longest
// chain, so the number of rounds is the hop-count critical path graham_para
// needs. With FWD and `lower`, also the weighted critical path of
// lower_bound (analysis.cpp:11-24, 72-81). Returns rounds, or -1 on a cycle,
// or -2 on overflow.
template <int W, class T, bool FWD>
K1_PHASE int p_closure(WarpState<W, T>& S, const int lane, const int n, bool lower,
                                      const PlatT<T> P) {
    bool ovf = false;
    bool flat = FWD && lower;  // every weight is t_min: the path is (hop length) x t_min
    if (FWD && lower) {
#pragma unroll 1
        for (int v = lane; v < n; v += 32) {
            const RatT<T> w = n_exec(RatT<T>{S.ln[v], S.ld[v]}, min(S.mmax[v], P.M), P);
            ovf |= w.d == 0;
            flat &= w.n == P.tmin.n && w.d == P.tmin.d;
            S.cn[v] = w.n;  // weight; replaced by the path prefix below
            S.cd[v] = w.d;
        }
        __syncwarp();
    }
    flat = __all_sync(FULL, flat);
    lower = lower && !flat;  // the weighted prefix is only needed when weights differ
    Mask<W> done;
    done.clear();
    int rounds = 0;
#pragma unroll 1
    for (;;) {
        const Mask<W> R = ballot_nodes<W>(lane, n, [&](int v) {
            if (v >= n || done.test(v)) return false;
            bool ok = true;
#pragma unroll
            for (int k = 0; k < W; ++k) ok &= ((FWD ? S.pred[v][k] : S.succ[v][k]) & ~done.w[k]) == 0;
            return ok;
        });
        if (!R.any()) break;
        ++rounds;
#pragma unroll 1
        for (int v = lane; v < n; v += 32) {
            if (!R.test(v)) continue;
            u64 a[W];
#pragma unroll
            for (int k = 0; k < W; ++k) a[k] = 0;
            RatT<T> best{0, 1};
            const Mask<W> pm = load_mask<W>(FWD ? S.pred[v] : S.succ[v]);
            for_bits<W>(pm, [&](int p) {
#pragma unroll
                for (int k = 0; k < W; ++k) a[k] |= FWD ? S.anc[p][k] : S.desc[p][k];
                a[p >> 6] |= 1ull << (p & 63);
                if (FWD && lower) {
                    const RatT<T> c{S.cn[p], S.cd[p]};
                    if (q_cmp(c, best) > 0) best = c;
                }
            });
#pragma unroll
            for (int k = 0; k < W; ++k) {
                if (FWD) S.anc[v][k] = a[k];
                else S.desc[v][k] = a[k];
            }
            if (FWD && lower) {
                const RatT<T> c = n_add(best, RatT<T>{S.cn[v], S.cd[v]});
                ovf |= c.d == 0;
                S.cn[v] = c.n;
                S.cd[v] = c.d;
            }
        }
#pragma unroll
        for (int k = 0; k < W; ++k) done.w[k] |= R.w[k];
        __syncwarp();
    }
    if (__any_sync(FULL, ovf)) return -2;
    return done.popc() == n ? (rounds | (flat ? kFlatPath : 0)) : -1;
}

// 32x32 bit-matrix transpose across a warp: lane i holds row i (bit c =
// element (i, c)); afterwards lane j holds column j. Five butterfly steps, each
// swapping the off-diagonal j x j blocks between lanes i and i ^ j.
__device__ __forceinline__ u32 warp_transpose32(u32 x, const int lane) {
    constexpr u32 m0[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int j = 16 >> s;
        const u32 y = __shfl_xor_sync(FULL, x, j);
        x = (lane & j) ? ((x & ~m0[s]) | ((y >> j) & m0[s])) : ((x & m0[s]) | ((y << j) & ~m0[s]));
    }
    return x;
}

// Descendants for n <= 64 as the transpose of the ancestor matrix:
// desc[v] = { u : v in anc[u] } — one to four 32x32 warp transposes replace the
// reverse Kahn rounds (dag.cpp:119-124).
template <class T>
K1_PHASE void p_desc_transpose(WarpState<1, T>& S, const int lane, const int n) {
    const u64 a0 = lane < n ? S.anc[lane][0] : 0ull;
    if (n <= 32) {
        const u32 t = warp_transpose32(u32(a0), lane);
        if (lane < n) S.desc[lane][0] = t;
    } else {
        const u64 a1 = lane + 32 < n ? S.anc[lane + 32][0] : 0ull;
        const u32 t00 = warp_transpose32(u32(a0), lane), t10 = warp_transpose32(u32(a1), lane);
        const u32 t01 = warp_transpose32(u32(a0 >> 32), lane), t11 = warp_transpose32(u32(a1 >> 32), lane);
        S.desc[lane][0] = (u64(t10) << 32) | t00;
        if (lane + 32 < n) S.desc[lane + 32][0] = (u64(t11) << 32) | t01;
    }
    __syncwarp();
}

// dag.cpp:97-108: exactly one source and one sink.
template <int W, class T>
K1_PHASE int p_ends(WarpState<W, T>& S, const int lane, const int n) {
    const Mask<W> src = ballot_nodes<W>(lane, n, [&](int v) {
        if (v >= n) return false;
        u64 a = 0;
#pragma unroll
        for (int k = 0; k < W; ++k) a |= S.pred[v][k];
        return a == 0;
    });
    if (src.popc() != 1) return DS_E_SOURCES;
    const Mask<W> snk = ballot_nodes<W>(lane, n, [&](int v) {
        if (v >= n) return false;
        u64 a = 0;
#pragma unroll
        for (int k = 0; k < W; ++k) a |= S.succ[v][k];
        return a == 0;
    });
    if (snk.popc() != 1) return DS_E_SINKS;
    return DS_OK;
}

// ------------------------------------------------------------- phase: bounds
// analysis.cpp:40-81 — greedy, greedy_unaware, graham_para, lower_bound.
template <int W, class T>
K1_PHASE int p_bounds(WarpState<W, T>& S, const int lane, const int n, const int closure,
                                     const PlatT<T> P, const u32 mask) {
    const int rounds = closure & (kFlatPath - 1);
    const bool flat = closure & kFlatPath;
    RatT<T> g{0, 1}, gu{0, 1}, tot{0, 1}, cp{0, 1};
    T units = 0;
    bool ovf = false;
    // integer operands add inline; only a fractional operand takes the call
    auto acc = [&](RatT<T>& s, const RatT<T> x) {
        if (s.d == 1 && x.d == 1) s.n = addc(s.n, x.n, ovf);
        else s = n_add(s, x);
    };
#pragma unroll 1
    for (int v = lane; v < n; v += 32) {
        const RatT<T> l{S.ln[v], S.ld[v]};
        // greedy's per-node time exec(l, min(m^max, M)) is the lower-bound
        // weight: when every one is t_min (flat) greedy is n * t_min
        if ((mask & DS_M_GREEDY) && !flat) acc(g, n_exec(l, min(S.mmax[v], P.M), P));
        if (mask & DS_M_GREEDY_UNAWARE) {
            acc(gu, S.mmax[v] <= P.M && flat ? P.tmin : n_exec(l, S.mmax[v], P));
        }
        if (mask & DS_M_GRAHAM_PARA) {  // ceil(load / t_min) unit nodes
            T u;
            if (P.tmin.n == 1 && P.tmin.d == 1 && l.d == 1) {
                u = l.n;
            } else {
                const RatT<T> q = n_div(l, P.tmin);
                ovf |= q.d == 0;
                u = n_ceil(q);
            }
            units = addc(units, u, ovf);
        }
        if (mask & DS_M_LOWER) {
            acc(tot, l);
            if (!flat) {
                const RatT<T> c{S.cn[v], S.cd[v]};
                if (n_cmp(c, cp) > 0) cp = c;
            }
        }
    }
    ovf |= g.d == 0 || gu.d == 0 || tot.d == 0;
#pragma unroll 1
    for (int o = 16; o; o >>= 1) {
        if ((mask & DS_M_GREEDY) && !flat) acc(g, RatT<T>{shfl_xor_w(g.n, o), shfl_xor_w(g.d, o)});
        if (mask & DS_M_GREEDY_UNAWARE) acc(gu, RatT<T>{shfl_xor_w(gu.n, o), shfl_xor_w(gu.d, o)});
        if (mask & DS_M_LOWER) acc(tot, RatT<T>{shfl_xor_w(tot.n, o), shfl_xor_w(tot.d, o)});
        units = addc(units, shfl_xor_w(units, o), ovf);
        if (!flat) {
            const RatT<T> c{shfl_xor_w(cp.n, o), shfl_xor_w(cp.d, o)};
            if (n_cmp(c, cp) > 0) cp = c;
        }
    }
    if ((mask & DS_M_GREEDY) && flat) g = n_mul_int(P.tmin, T(n));
    ovf |= g.d == 0 || gu.d == 0 || tot.d == 0;
    if (lane == 0) {
        if (mask & DS_M_GREEDY) {
            S.bn[DS_BOUND_GREEDY] = g.n;
            S.bd[DS_BOUND_GREEDY] = g.d;
        }
        if (mask & DS_M_GREEDY_UNAWARE) {
            S.bn[DS_BOUND_GREEDY_UNAWARE] = gu.n;
            S.bd[DS_BOUND_GREEDY_UNAWARE] = gu.d;
        }
        if (mask & DS_M_GRAHAM_PARA) {
            // chain = (longest hop path) * t_min; bound = chain + (work - chain) / M
            const RatT<T> work = n_mul_int(P.tmin, units);
            const RatT<T> chain = n_mul_int(P.tmin, T(rounds));
            const RatT<T> r = n_add(chain, n_div_int(n_sub(work, chain), T(P.M)));
            ovf |= work.d == 0 || chain.d == 0 || r.d == 0;
            S.bn[DS_BOUND_GRAHAM_PARA] = r.n;
            S.bd[DS_BOUND_GRAHAM_PARA] = r.d;
        }
        if (mask & DS_M_LOWER) {
            const RatT<T> wf = n_div_int(tot, T(P.M));
            ovf |= wf.d == 0;
            if (flat) {  // all weights t_min: critical path = hop length x t_min
                cp = n_mul_int(P.tmin, T(rounds));
                ovf |= cp.d == 0;
            }
            const RatT<T> r = n_cmp(wf, cp) < 0 ? cp : wf;
            S.bn[DS_BOUND_LOWER] = r.n;
            S.bd[DS_BOUND_LOWER] = r.d;
        }
    }
    __syncwarp();
    return __any_sync(FULL, ovf) ? DS_EOVERFLOW : DS_OK;
}

// --------------------------------------------------------- phase: W^anc, ranks
// dag.cpp:126-135 W^anc = load + sum of ancestors' loads; ranks in
// (W^anc desc, id asc) for heads (division.cpp:88-93) and candidates
// (scheduler.cpp:275-280); joins in (W^anc asc, id asc) (dag.cpp:218-230).
// Returns the join count, or -1 on overflow.
template <int W, class T>
K1_PHASE int p_rank(WarpState<W, T>& S, const int lane, const int n, const bool integer) {
    bool ovf = false;
#pragma unroll 1
    for (int v = lane; v < n; v += 32) {
        const Mask<W> am = load_mask<W>(S.anc[v]);
        if (integer) {
            T s = S.ln[v];
            for_bits<W>(am, [&](int u) { s = addc(s, S.ln[u], ovf); });
            S.xn[v] = s;
            S.xd[v] = 1;
        } else {
            RatT<T> s{S.ln[v], S.ld[v]};
            for_bits<W>(am, [&](int u) { s = n_add(s, RatT<T>{S.ln[u], S.ld[u]}); });
            ovf |= s.d == 0;
            S.xn[v] = s.n;
            S.xd[v] = s.d;
        }
    }
    __syncwarp();
    const Mask<W> J = ballot_nodes<W>(lane, n, [&](int v) {
        if (v >= n) return false;
        int c = 0;
#pragma unroll
        for (int k = 0; k < W; ++k) c += __popcll(S.pred[v][k]);
        return c >= 2;
    });
    if constexpr (W == 1) {
        // Integer W^anc (the common case): two warp bitonic sorts of 64 keys
        // (2 per lane) replace the O(n) compare loop per node. Key for the
        // rank: (W^anc desc, id asc) = ((~W) << 8 | id); for the joins:
        // (W^anc asc, id asc) = (W << 8 | id), non-joins pushed to the end.
        // Keys fit 32 bits (W^anc < 2^24, the C5 case) or 64 (W^anc < 2^48).
        u64 wmax = 0;
        for (int v = lane; v < n; v += 32) wmax = max(wmax, u64(S.xn[v]));
        const u32 whi = __reduce_max_sync(FULL, u32(wmax >> 32)), wlo = __reduce_max_sync(FULL, u32(wmax));
        wmax = whi ? (u64(whi) << 32 | 0xffffffffull) : u64(wlo);  // an upper bound is enough
        if (integer && wmax < (1ull << 48)) {
            const bool k32 = wmax < (1ull << 24);
            auto sort_keys = [&](auto kz) {
                using K_t = decltype(kz);
                const K_t top = k32 ? K_t((1u << 24) - 1) : K_t((1ull << 48) - 1), none = ~K_t(0);
                K_t a = lane < n ? ((top - K_t(S.xn[lane])) << 8) | K_t(lane) : none;
                K_t b = lane + 32 < n ? ((top - K_t(S.xn[lane + 32])) << 8) | K_t(lane + 32) : none;
                K_t ja = lane < n && J.test(lane) ? (K_t(S.xn[lane]) << 8) | K_t(lane) : none;
                K_t jb = lane + 32 < n && J.test(lane + 32) ? (K_t(S.xn[lane + 32]) << 8) | K_t(lane + 32) : none;
                bitonic64x2<K_t>(a, b, ja, jb, lane, n <= 32 ? 32 : 64);
                if (a != none) {
                    S.order[lane] = short(a & 0xff);
                    S.rank[a & 0xff] = short(lane);
                }
                if (b != none) {
                    S.order[lane + 32] = short(b & 0xff);
                    S.rank[b & 0xff] = short(lane + 32);
                }
                if (ja != none) S.jorder[lane] = short(ja & 0xff);
                if (jb != none) S.jorder[lane + 32] = short(jb & 0xff);
            };
            if (k32) sort_keys(u32(0));
            else sort_keys(u64(0));
            __syncwarp();
            if (__any_sync(FULL, ovf)) return -1;
            return J.popc();
        }
    }
#pragma unroll 1
    for (int v = lane; v < n; v += 32) {
        const RatT<T> wv{S.xn[v], S.xd[v]};
        int r = 0, jr = 0;
        const bool isj = J.test(v);
#pragma unroll 1
        for (int u = 0; u < n; ++u) {
            int c;
            if (integer) c = S.xn[u] < wv.n ? -1 : (S.xn[u] > wv.n ? 1 : 0);
            else c = q_cmp(RatT<T>{S.xn[u], S.xd[u]}, wv);
            r += (c > 0) || (c == 0 && u < v);
            jr += isj && J.test(u) && ((c < 0) || (c == 0 && u < v));
        }
        S.rank[v] = short(r);
        S.order[r] = short(v);
        if (isj) S.jorder[jr] = short(v);
    }
    __syncwarp();
    if (__any_sync(FULL, ovf)) return -1;
    return J.popc();
}

// ----------------------------------------------------------- phase: division
// division.cpp:10-30 blocks in join order + residual; :67-126 groups.
template <int W, class T, bool DETAIL>
K1_PHASE int p_division(WarpState<W, T>& S, const int lane, const int n, const int n_joins,
                                       const int M, DetailOut det) {
    Mask<W> V, assigned;
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int lo = k * 64;
        V.w[k] = n >= lo + 64 ? ~0ull : (n <= lo ? 0ull : ((1ull << (n - lo)) - 1));
    }
    assigned.clear();
    const Mask<W> big = ballot_nodes<W>(lane, n, [&](int v) { return v < n && S.mmax[v] >= M; });
    int n_div = 0;
#pragma unroll 1
    for (int b = 0; b <= n_joins; ++b) {
        Mask<W> B;
        if (b < n_joins) {
            const int th = S.jorder[b];
#pragma unroll
            for (int k = 0; k < W; ++k) B.w[k] = S.anc[th][k] & ~assigned.w[k];
        } else {
#pragma unroll
            for (int k = 0; k < W; ++k) B.w[k] = V.w[k] & ~assigned.w[k];
        }
#pragma unroll
        for (int k = 0; k < W; ++k) assigned.w[k] |= B.w[k];
        if (DETAIL) {
#pragma unroll 1
            for (int v = lane; v < n; v += 32) {
                if (B.test(v)) det.node_block[v] = short(b);
            }
        }
        Mask<W> grouped;
        grouped.clear();
#pragma unroll 1
        while (!grouped.eq(B)) {  // empty blocks are skipped (division.cpp:73)
            // heads: ungrouped members whose in-block predecessor is grouped or absent
            const Mask<W> H = ballot_nodes<W>(lane, n, [&](int v) {
                if (v >= n || !B.test(v) || grouped.test(v)) return false;
                bool ok = true;
#pragma unroll
                for (int k = 0; k < W; ++k) ok &= (S.pred[v][k] & B.w[k] & ~grouped.w[k]) == 0;
                return ok;
            });
            if (!H.any()) break;
            Mask<W> sel = H;
            if (H.popc() > M) {  // Rule 1: keep the top-M by rank
#pragma unroll
                for (int k = 0; k < W; ++k) S.rmask[k] = 0;
                __syncwarp();
#pragma unroll 1
                for (int v = lane; v < n; v += 32) {
                    if (H.test(v)) smem_set_bit(S.rmask, S.rank[v]);
                }
                __syncwarp();
                sel = ballot_nodes<W>(lane, n, [&](int v) {
                    if (v >= n || !H.test(v)) return false;
                    const int r = S.rank[v];
                    int below = 0;
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        const u64 w = S.rmask[k];
                        if (k * 64 + 64 <= r) below += __popcll(w);
                        else if (k * 64 < r) below += __popcll(w & ((1ull << (r - k * 64)) - 1));
                    }
                    return below < M;
                });
                __syncwarp();
            }
            // Rule 2: any selected head with m^max >= M -> the max-m^max head
            // alone (only a question when several heads and an oversized one)
            Mask<W> sb;
#pragma unroll
            for (int k = 0; k < W; ++k) sb.w[k] = sel.w[k] & big.w[k];
            if (sb.any() && sel.popc() > 1) {
                int mx = 0;
#pragma unroll 1
                for (int v = lane; v < n; v += 32) {
                    if (sb.test(v)) mx = max(mx, S.mmax[v]);
                }
                mx = __reduce_max_sync(FULL, mx);
                const Mask<W> top = ballot_nodes<W>(lane, n, [&](int v) {
                    return v < n && sb.test(v) && S.mmax[v] == mx;
                });
                int pick = -1;
#pragma unroll
                for (int k = W - 1; k >= 0; --k) {
                    if (top.w[k]) pick = k * 64 + __ffsll(top.w[k]) - 1;
                }
                sel.clear();
                sel.set(pick);
            }
#pragma unroll
            for (int k = 0; k < W; ++k) {
                grouped.w[k] |= sel.w[k];
                S.divg[n_div][k] = sel.w[k];
            }
            if (DETAIL) {
#pragma unroll 1
                for (int v = lane; v < n; v += 32) {
                    if (sel.test(v)) det.node_div_group[v] = short(n_div);
                }
            }
            ++n_div;
        }
    }
    __syncwarp();
    return n_div;
}

template <class T>
__device__ __forceinline__ void put_rec(ds_entity_rec& e, int origin, int gen, int part, bool launched, int group,
                                        int m, RatT<T> load, RatT<T> exec, RatT<T> res, bool& ovf) {
    e.origin = (unsigned short)origin;
    e.generation = (unsigned short)gen;
    e.part = (unsigned char)part;
    e.launched = launched ? 1 : 0;
    e.group = (unsigned short)group;
    e.parallelism = m;
    e.reserved = 0;
    ovf |= !fits_i64(load.n) || !fits_i64(load.d) || !fits_i64(exec.n) || !fits_i64(exec.d) ||
           !fits_i64(res.n) || !fits_i64(res.d);
    e.load_num = (long long)load.n;
    e.load_den = (long long)load.d;
    e.exec_num = (long long)exec.n;
    e.exec_den = (long long)exec.d;
    e.res_num = (long long)res.n;
    e.res_den = (long long)res.d;
}

// ------------------------------------------------- apportion member selection
// shed: min k1, ties smaller index (scheduler.cpp:60-72); fill: max k1, then
// max k2, ties smaller index (:74-93).
template <class T>
struct Pick {
    RatT<T> k1, k2;
    int idx;
};
template <class T>
__device__ __forceinline__ bool pick_better(const Pick<T>& a, const Pick<T>& b, const bool shed) {
    if (a.idx < 0) return false;
    if (b.idx < 0) return true;
    int c = q_cmp(a.k1, b.k1);
    if (shed) c = -c;
    if (c == 0) c = q_cmp(a.k2, b.k2);  // shed: k2 is constant
    return c > 0 || (c == 0 && a.idx < b.idx);
}
// ----------------------------------------------------------- phase: schedule
// scheduler.cpp:214-359, one executed group per non-absorbed division group.
// Returns status | (n_groups << 8) | (n_entities << 20).
template <int W, class T, bool DETAIL>
K1_PHASE long long p_schedule(WarpState<W, T>& S, const int lane, const int n, const int n_div,
                                             const PlatT<T> P, DetailOut det) {
    bool ovf = false;
    Mask<W> V;
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int lo = k * 64;
        V.w[k] = n >= lo + 64 ? ~0ull : (n <= lo ? 0ull : ((1ull << (n - lo)) - 1));
    }
    RatT<T> proposed{0, 1};
    int gidx = 0, n_ent = 0;
    Mask<W> done;
    done.clear();
#pragma unroll 1
    for (int g = 0; g < n_div; ++g) {
        const Mask<W> G = load_mask<W>(S.divg[g]);
        Mask<W> org;
#pragma unroll
        for (int k = 0; k < W; ++k) org.w[k] = G.w[k] & ~done.w[k];
        if (!org.any()) continue;  // fully absorbed by earlier launches

        // -- apportion (scheduler.cpp:35-95) over the pending loads
        RatT<T> R{0, 1};
        int used = 0, n_mem = 0, bott_pos = 0;
        const bool single = sizeof(T) < 16 && org.popc() == 1;
        if (single) {
            // one pending member (70% of C5 groups): quota = l*M/l = M, so
            // m = cap = min(m^max, M), no shed/fill, and it is the response
            int v = 0;
#pragma unroll
            for (int k = W - 1; k >= 0; --k) {
                if (org.w[k]) v = k * 64 + __ffsll(org.w[k]) - 1;
            }
            const RatT<T> l{S.pn[v], S.pd[v]};
            int cp = q_max_par(l, P);
            if (cp < 0) {
                ovf = true;
                cp = 1;
            }
            cp = min(cp, P.M);
            R = q_exec(l, cp, P);
            ovf |= R.d == 0;
            used = cp;
            n_mem = 1;
            if (DETAIL) {
                if (lane == 0) {
                    S.mq[v] = cp;
                    S.xn[v] = R.n;
                    S.xd[v] = R.d;
                }
                __syncwarp();
            }
        } else {
            RatT<T> Wt{0, 1};
            for_bits<W>(org, [&](int v) { Wt = q_add(Wt, RatT<T>{S.pn[v], S.pd[v]}); });
            ovf |= Wt.d == 0;
            int tot = 0, capsum = 0;
#pragma unroll 1
            for (int v = lane; v < n; v += 32) {
                if (!org.test(v)) continue;
                const RatT<T> l{S.pn[v], S.pd[v]};
                int cp = q_max_par(l, P);
                if (cp < 0) {
                    ovf = true;
                    cp = 1;
                }
                cp = min(cp, P.M);
                // quota = l*M/W = (l.n*M*W.d) / (l.d*W.n); floor and remainder
                const T qn = mulc(mulc(l.n, T(P.M), ovf), Wt.d, ovf);
                const T qd = mulc(l.d, Wt.n, ovf);
                const T fl = divw(qn, qd);
                const long long flc = fl > T(0x7fffffff) ? 0x7fffffffll : (long long)fl;
                const long long base = max(1ll, min(flc, (long long)cp));
                S.mq[v] = int(base);
                S.cap[v] = cp;
                S.rn[v] = qn - fl * qd;
                S.rd[v] = qd;
                tot += int(base);
                capsum += cp;
            }
            tot = __reduce_add_sync(FULL, tot);
            capsum = __reduce_add_sync(FULL, capsum);
            __syncwarp();
            // shed while over M (smallest slowdown exec(m-1), first index wins
            // ties), else fill up to target (largest exec(m), then larger remainder,
            // then first index); shedding ends at M >= target, so at most one runs
            const int target = min(P.M, capsum);
#pragma unroll 1
            while (tot > P.M || tot < target) {
                const bool shed = tot > P.M;
                Pick<T> c{{0, 1}, {0, 1}, -1};
                for_bits<W>(org, [&](int v) {
                    const int m = S.mq[v];
                    if (shed ? m <= 1 : m >= S.cap[v]) return;
                    const Pick<T> x{q_exec_raw(RatT<T>{S.pn[v], S.pd[v]}, shed ? m - 1 : m, P),
                                    shed ? RatT<T>{0, 1} : RatT<T>{S.rn[v], S.rd[v]}, v};
                    ovf |= x.k1.d == 0;
                    if (pick_better<T>(x, c, shed)) c = x;
                });
                if (c.idx < 0) return DS_EINVARIANT;
                const int step = shed ? -1 : 1;
                if (lane == 0) S.mq[c.idx] += step;
                __syncwarp();
                tot += step;
            }

            // -- members: exec, response (first strict max), bottleneck
#pragma unroll 1
            for (int v = lane; v < n; v += 32) {
                if (!org.test(v)) continue;
                const RatT<T> e = q_exec(RatT<T>{S.pn[v], S.pd[v]}, S.mq[v], P);
                ovf |= e.d == 0;
                S.xn[v] = e.n;
                S.xd[v] = e.d;
            }
            __syncwarp();
            int bott = -1;
            for_bits<W>(org, [&](int v) {
                const RatT<T> e{S.xn[v], S.xd[v]};
                if (bott < 0 || q_cmp(e, R) > 0) {
                    R = e;
                    bott = v;
                    bott_pos = n_mem;
                }
                used += S.mq[v];
                ++n_mem;
            });
        }
        const int spare0 = P.M - used;

        // -- candidates (scheduler.cpp:253-280). Concurrency is symmetric, so
        // the pool is the union of the members' concurrent sets minus the
        // division group (which also removes each member itself).
        Mask<W> pool;
        if constexpr (W == 1) {
            // lanes OR their members' concurrent sets, the warp reduces (REDUX)
            u64 c = 0;
            if (org.test(lane)) c = ~(S.anc[lane][0] | S.desc[lane][0]);
            if (lane + 32 < n && org.test(lane + 32)) c |= ~(S.anc[lane + 32][0] | S.desc[lane + 32][0]);
            pool.w[0] = V.w[0] & ((u64(__reduce_or_sync(FULL, u32(c >> 32))) << 32) | __reduce_or_sync(FULL, u32(c)));
        } else {
            pool.clear();
            for_bits<W>(org, [&](int v) {
#pragma unroll
                for (int k = 0; k < W; ++k) pool.w[k] |= V.w[k] & ~(S.anc[v][k] | S.desc[v][k]);
            });
        }
        Mask<W> avail;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            pool.w[k] &= ~G.w[k];
            avail.w[k] = pool.w[k] & ~done.w[k];
        }
        Mask<W> cands;
        cands.clear();
        if (avail.any() && (DETAIL || spare0 >= 1)) {
            cands = ballot_nodes<W>(lane, n, [&](int c) {
                if (c >= n || !avail.test(c)) return false;
                bool ok = true;
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    ok &= (S.pred[c][k] & pool.w[k]) == 0;   // a source of the pool
                    ok &= (S.pred[c][k] & ~done.w[k]) == 0;  // released: preds done earlier
                }
                return ok;
            });
        }

        // -- launches in rank order (scheduler.cpp:286-330)
        Mask<W> whole;
        whole.clear();
        int spare = spare0, n_launch = 0;
        const int first_ent = n_ent;
        if (cands.any() && spare >= 1) {
#pragma unroll
            for (int k = 0; k < W; ++k) S.rmask[k] = 0;
            __syncwarp();
#pragma unroll 1
            for (int v = lane; v < n; v += 32) {
                if (cands.test(v)) smem_set_bit(S.rmask, S.rank[v]);
            }
            __syncwarp();
            const Mask<W> rm = load_mask<W>(S.rmask);
            bool stop = false;
            for_bits<W>(rm, [&](int r) {
                if (stop) return;
                if (spare < 1) {
                    stop = true;
                    return;
                }
                const int c = S.order[r];
                const RatT<T> l{S.pn[c], S.pd[c]};
                int mp = q_max_par(l, P);
                if (mp < 0) {
                    ovf = true;
                    mp = 1;
                }
                const int mc = min(mp, spare);
                const RatT<T> dur = q_exec(l, mc, P);
                ovf |= dur.d == 0;
                if (q_cmp(dur, R) <= 0) {
                    if (DETAIL && lane == 0) {
                        put_rec(det.ent[n_ent], c, S.gen[c], S.ppart[c], true, gidx, mc, l, dur, RatT<T>{0, 0},
                                ovf);
                    }
                    whole.set(c);
                    spare -= mc;
                } else {
                    const RatT<T> pl = n_mul_int(R, T(mc));
                    const RatT<T> rl = n_sub(l, pl);
                    ovf |= pl.d == 0 || rl.d == 0;
                    const int gn = S.gen[c] + 1;
                    if (DETAIL && lane == 0) put_rec(det.ent[n_ent], c, gn, 1, true, gidx, mc, pl, R, rl, ovf);
                    __syncwarp();
                    if (lane == 0) {
                        S.gen[c] = (unsigned short)gn;
                        S.ppart[c] = 2;
                        S.pn[c] = rl.n;
                        S.pd[c] = rl.d;
                    }
                    spare -= mc;
                    stop = true;
                }
                ++n_ent;
                ++n_launch;
                __syncwarp();
            });
        }

        // -- commit members (scheduler.cpp:348-356)
        if (DETAIL) {
            int pos = 0;
            for_bits<W>(org, [&](int v) {
                if (lane == 0) {
                    put_rec(det.ent[n_ent + pos], v, S.gen[v], S.ppart[v], false, gidx, S.mq[v],
                            RatT<T>{S.pn[v], S.pd[v]}, RatT<T>{S.xn[v], S.xd[v]}, RatT<T>{0, 0}, ovf);
                }
                ++pos;
            });
            if (lane == 0) {
                ds_group_rec& gr = det.grp[gidx];
                ovf |= !fits_i64(R.n) || !fits_i64(R.d);
                gr.resp_num = (long long)R.n;
                gr.resp_den = (long long)R.d;
                gr.spare_sms = spare0;
                gr.div_group = (unsigned short)g;
                gr.bottleneck = (unsigned short)(first_ent + n_launch + bott_pos);
                gr.first_entity = (unsigned short)first_ent;
                gr.n_launches = (unsigned short)n_launch;
                gr.n_members = (unsigned short)n_mem;
                gr.reserved = 0;
                if (det.unl) {
                    for (int k = 0; k < det.unl_w; ++k) det.unl[gidx * det.unl_w + k] = cands.w[k] & ~whole.w[k];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < W; ++k) done.w[k] |= org.w[k] | whole.w[k];
        n_ent += n_mem;
        proposed = q_add(proposed, R);
        ovf |= proposed.d == 0;
        ++gidx;
        __syncwarp();
    }
    if (!done.eq(V)) return DS_EINVARIANT;  // "scheduling finished with unplaced kernels"
    if (lane == 0) {
        S.bn[DS_BOUND_PROPOSED] = proposed.n;
        S.bd[DS_BOUND_PROPOSED] = proposed.d;
    }
    __syncwarp();
    const int st = __any_sync(FULL, ovf) ? DS_EOVERFLOW : DS_OK;
    return (long long)st | ((long long)gidx << 8) | ((long long)n_ent << 20);
}

// -------------------------------------------------------------- one DAG
// Returns status; fills S.bn/S.bd and the out-params.
template <int W, class T, bool DETAIL, bool FRONT = false>
__device__ __forceinline__ int analyse_dag(WarpState<W, T>& S, const int lane, const int n,
                                           const u64* __restrict__ lnum, const u64* __restrict__ lden,
                                           const u32* __restrict__ edges, const int n_edges, const PlatT<T> P,
                                           const u32 mask, int& n_groups, DetailOut det, int& n_ent, int& n_div) {
    constexpr int N = WarpState<W, T>::N;
    n_groups = 0;
    n_ent = 0;
    n_div = 0;
    if (lane < DS_N_BOUNDS) {
        S.bn[lane] = 0;
        S.bd[lane] = 0;
    }
    if (n <= 0) return DS_E_EMPTY;
    if (n > N) return DS_ETOOBIG;
    int st = p_load<W, T>(S, lane, n, lnum, lden, P);
    if ((st & 0xff) != DS_OK) return st & 0xff;
    const bool integer = (st >> 8) & 1;
    const bool low_t = (st >> 9) & 1;
    __syncwarp();
    if ((st = p_edges<W, T>(S, lane, n, edges, n_edges)) != DS_OK) return st;
    const bool lower = mask & DS_M_LOWER;
    const int closure = p_closure<W, T, true>(S, lane, n, lower, P);
    if (closure == -1) return DS_E_CYCLE;
    if (closure == -2) return DS_EOVERFLOW;
    const int rounds = closure;  // hop count | kFlatPath, decoded by p_bounds
    if ((st = p_ends<W, T>(S, lane, n)) != DS_OK) return st;
    // DagTask::make succeeded; method_bound(proposed) comes first in
    // evaluate_corpus's order and schedule() throws on a load below t_min
    // (detail mode still forms the division first: build_groups has no such
    // check, division.cpp:67-126)
    if (low_t && (mask & DS_M_PROPOSED) && !DETAIL) return DS_E_LOAD_TMIN;
    if constexpr (W == 1) p_desc_transpose<T>(S, lane, n);
    else p_closure<W, T, false>(S, lane, n, false, P);
    if (mask & (DS_M_GREEDY | DS_M_GREEDY_UNAWARE | DS_M_GRAHAM_PARA | DS_M_LOWER)) {
        if ((st = p_bounds<W, T>(S, lane, n, rounds, P, mask)) != DS_OK) return st;
    }
    if (FRONT || !((mask & DS_M_PROPOSED) || DETAIL)) return DS_OK;  // FRONT: k1_mid, k1_back go on
    const int n_joins = p_rank<W, T>(S, lane, n, integer);
    if (n_joins < 0) return DS_EOVERFLOW;
    n_div = p_division<W, T, DETAIL>(S, lane, n, n_joins, P.M, det);
    if (DETAIL && low_t) return DS_E_LOAD_TMIN;
    const long long r = p_schedule<W, T, DETAIL>(S, lane, n, n_div, P, det);
    n_groups = int((r >> 8) & 0xfff);
    n_ent = int(r >> 20);
    return int(r & 0xff);
}

#ifndef DS_SORT_WINDOW
#define DS_SORT_WINDOW 4096
#endif
constexpr u64 kSortWindow = DS_SORT_WINDOW;  // DAGs per walk-order sort window (0: global)

// Three-kernel split of the 32-bit W=1 bounds pass. As one kernel it is
// instruction-fetch bound (its hot code exceeds the SM's 32 KB L1.5
// instruction cache; ncu: ~60% of stall samples "no_instructions"), so it runs
// as k1_front (load, edges, closure, ends, descendants, bounds), k1_mid (ranks,
// division) and k1_back (schedule), each with a hot loop that fits, over
// per-node state left in HBM (~42 B per node, written and re-read once).
// Status codes mark the hand-over.
constexpr int32_t kStMid = -999;       // k1_front done, k1_mid pending
constexpr int32_t kStPending = -1000;  // k1_mid done, k1_back pending
constexpr int32_t kStRetried = -1001;  // queued for a wider tier
// Per node, what k1_back reads from k1_front, in one 32-byte record (one
// sector, written whole so L2 never has to fill it from DRAM): the
// one-lane-per-DAG walk touches a node's pred, anc|desc and load together, so
// a record costs it one line where three arrays cost three. k1_mid's
// rank/order goes to its own array (a 2-byte update of the record would make
// every sector dirty again).
struct K1Node {
    u64 pred;
    u64 ad;          // anc | desc: the complement of v's concurrent set (+ v)
    u32 ln, ld;      // canonical load
    u64 pad;
};
static_assert(sizeof(K1Node) == 32, "K1Node is one sector");
// Compact hand-off of a DAG with n <= 32 nodes and integer loads (k1_fast<32>):
// per node a 16-byte record (u32 masks, load, rank | order << 8), then one u32
// member mask per division group, all inside the DAG's own 32n-byte slice of
// the K1Node array — 16n + 4 ndiv bytes in one contiguous run instead of 32n +
// 2n + 8 ndiv over three arrays, so a lane's walk touches ~half the lines.
// h.ndiv[d] carries kNdivCompact to say which layout a DAG has.
struct K1Rec16 {
    u32 pred;
    u32 ad;  // anc | desc
    u32 ln;  // integer load (den 1)
    u32 ro;  // rank | order << 8
};
static_assert(sizeof(K1Rec16) == 16, "K1Rec16 is 16 bytes");
constexpr uint16_t kNdivCompact = 0x8000;
// Walk-order sort key (52 bits; k1_wsort appends the 12-bit window index):
// the hand-off layout first (a warp's lanes then read one layout), then the
// division-group shape. Called by every lane of the warp with c = the member
// count of division group `lane` and c2 = that of group lane + 32 (0 when
// absent). mode (K1Args::key_mode, DS_WALK_KEY):
//   0  group count (6 bits) + member counts clipped to 3 of groups 0..9
//   1  group count (5 bits) + member counts clipped to 3 of groups 0..22
//   2  group count (5 bits) + one "several members" bit for groups 0..45
__device__ __forceinline__ u64 walk_key(const int lane, const u32 ndiv, const u32 c, const u32 c2, const bool compact,
                                        const int mode) {
    const u64 top = (compact ? 0ull : 1ull) << 51;
    if (mode == 1) {
        const u32 f = lane < 23 ? min(c, 3u) : 0u;
        const int sh = 2 * (22 - min(lane, 22));  // group g at bits 45-2g..44-2g
        const u32 lo = __reduce_or_sync(FULL, sh < 32 ? f << sh : 0u);
        const u32 hi = __reduce_or_sync(FULL, sh >= 32 ? f << (sh - 32) : 0u);
        return top | (u64(min(ndiv, 31u)) << 46) | (u64(hi) << 32) | lo;
    }
    if (mode == 2) {
        const u32 b1 = __ballot_sync(FULL, c >= 2), b2 = __ballot_sync(FULL, lane < 14 && c2 >= 2);
        // group g at bit 45-g
        const u64 bits = (u64(__brev(b1)) << 14) | (u64(__brev(b2) >> 18) & 0x3fffull);
        return top | (u64(min(ndiv, 31u)) << 46) | bits;
    }
    const u32 f = lane < 10 ? min(c, 3u) : 0u;
    const u32 shape = (min(ndiv, 63u) << 20) | __reduce_or_sync(FULL, f << (18 - 2 * min(lane, 9)));
    return top | shape;
}
constexpr int kDefaultWalkKey = 0;
// Smallest compact walk key with at least `groups` division groups (the
// group count sits above the shape bits: bits 20-25 in layout 0, 46-50 in
// layouts 1 and 2) — the heavy class of k1_back_lane's task order.
// DS_K1_HEAVY_GROUPS overrides the default of 15 (C5: 14.5 groups per DAG).
inline u64 walk_key_heavy(int mode) {
    static const u64 groups = [] {
        const char* env = getenv("DS_K1_HEAVY_GROUPS");
        const long v = env ? atol(env) : 15;
        return u64(v >= 0 && v < 64 ? v : 15);
    }();
    return mode == 0 ? (groups << 20) : (std::min<u64>(groups, 31) << 46);
}
constexpr u64 kWalkKeyNone = ~0ull;  // never walked (k1_fast left it to the general kernels)
struct K1Handoff {   // over the batch's node index (node_off[d] - node_off[0] + v)
    K1Node* node;
    u64* anc;        // k1_mid's block construction
    u64* divg;       // division group g of DAG d at node slot g
    uint16_t* ro;    // rank[v] | order[v] << 8 (k1_mid)
    uint16_t* ndiv;  // per DAG
    // walk order for k1_back_lane: k1_mid keys every DAG by its shape (group
    // count, which division groups have several members), k1_wsort orders
    // the DAG indices by it within windows of kSortWindow DAGs, and the lanes
    // of a warp then walk DAGs that take the same branches
    u64* skey;       // per DAG: walk-order key (k1_fast / k1_mid), walk_key()
    u32* perm;       // walk order out of k1_wsort
    u32* fb;         // DAGs k1_fast left to the general kernels (count: retry_count[7])
    u32* l64;        // DAGs with 32 < n <= 64 for k1_fast<64> (count: retry_count[8])
    u32* wcnt;       // per sort window: walked light compact / heavy compact / wide DAGs (k1_wsort)
};

// The triangular wire form (ds_dag_batch_tri) as K1 reads it: the fast path
// takes each node's predecessor mask straight out of the adjacency bits; the
// wide arrays (u64 loads, capacity-layout edge list) are written on demand
// for the DAGs the general kernels take (k1_tri.cuh).
struct TriWire {
    const u32* adj = nullptr;       // strictly lower-triangular bits, node v's preds at v(v-1)/2 ..
    const u32* adj_off = nullptr;   // [n + 1] word offsets (relative to adj_off[0])
    const uint16_t* ln16 = nullptr; // [N] integer loads
    u64* ln = nullptr;              // widened: the K1Args::load_num array
    u32* edge_off = nullptr;        // widened: K1Args::edge_off (32 edges per adjacency word)
    u32* edge_cnt = nullptr;        // widened: K1Args::edge_cnt
    u32* edges = nullptr;           // widened: K1Args::edges
};

// node v's predecessor mask (v < 64) from a DAG's triangular words w[0 .. nw)
__device__ __forceinline__ u64 tri_preds(const u32* w, u32 nw, int n, int v) {
    if (v <= 0 || v >= n) return 0;
    const u32 o = u32(v) * u32(v - 1) / 2, k = o >> 5, sh = o & 31;
    u64 x = w[k] >> sh;
    if (k + 1 < nw) x |= u64(w[k + 1]) << (32 - sh);
    if (sh && k + 2 < nw) x |= u64(w[k + 2]) << (64 - sh);
    return x & ((1ull << v) - 1);
}

struct K1Args {
    u64 n_dags;
    const u32* node_off;
    const u32* edge_off;
    const u64* load_num;
    const u64* load_den;
    const u32* edges;
    const u64* unl_base;   // detail mode: per DAG, its first word in det.unlaunched
    u32* big_q;            // n > 256: DAG indices queued from the 32- to the 64-bit
                           // tier ([0, n)) and from the 64- to the 128-bit tier
                           // ([n, 2n)); counts at retry_count[10], [11]
    unsigned char* big_scratch;  // n > 512: global-memory warp states (k1_big<16>)
    const u32* edge_cnt;   // optional per-DAG edge counts: DAG d's edges are
                           // edges[edge_off[d] ..][0 .. edge_cnt[d]) (capacity
                           // layout of the expanded triangular form)
    PlatT<u64> plat;
    u32 mask;
    int32_t* status;
    int64_t* bounds;
    uint16_t* n_groups;
    ds_scheme_out det;     // detail mode
    u32* retry;            // DAG indices whose 32-bit pass overflowed
    u32* retry_count;
    u32* retry2;           // ... and whose 64-bit pass overflowed
    u32* retry2_count;
    K1Handoff h;           // split mode when h.node != nullptr (bounds mode only)
    const u32* perm;       // k1_back_lane's DAG order (nullptr: index order)
    int fb_only;           // k1_front / k1_mid take only the DAGs k1_fast queued (h.fb)
    int key_mode;          // walk_key() layout (DS_WALK_KEY)
    TriWire tri;           // triangular wire form (tri.adj != nullptr)
};

template <int W, class T, bool DETAIL>
__device__ __forceinline__ void run_one(WarpState<W, T>& S, const int lane, const K1Args& a, const u64 d,
                                        const u32 nbase, const u32 ebase, const PlatT<T> P, u32* next,
                                        u32* next_count) {
    const u32 n0 = a.node_off[d] - nbase, n1 = a.node_off[d + 1] - nbase;
    const u32 e0 = a.edge_off[d] - ebase, e1 = a.edge_cnt ? e0 + a.edge_cnt[d] : a.edge_off[d + 1] - ebase;
    const int n = int(n1 - n0);
    int ng = 0, nent = 0, ndiv = 0;
    DetailOut det{};
    if (DETAIL) {
        det.ent = a.det.entities + 2ull * n0;
        det.grp = a.det.groups + n0;
        det.node_block = a.det.node_block + n0;
        det.node_div_group = a.det.node_div_group + n0;
        det.unl = a.det.unlaunched && a.unl_base ? a.det.unlaunched + a.unl_base[d] : nullptr;
        det.unl_w = (n + 63) / 64;
    }
    int st = analyse_dag<W, T, DETAIL>(S, lane, n, a.load_num + n0, a.load_den ? a.load_den + n0 : nullptr,
                                       a.edges + e0, int(e1 - e0), P, a.mask, ng, det, nent, ndiv);
    if (st == DS_EOVERFLOW && next) {
        // re-run in wider words (k1_analyse_retry); nothing is written now
        if (lane == 0) next[atomicAdd(next_count, 1u)] = u32(d);
        __syncwarp();
        return;
    }
    // canonical results must fit the ABI's int64 slots
    if (st == DS_OK) {
        bool fit = true;
        if (lane < DS_N_BOUNDS) fit = fits_i64(S.bn[lane]) && fits_i64(S.bd[lane]);
        if (!__all_sync(FULL, fit)) st = DS_EOVERFLOW;
    }
    int64_t* b = (DETAIL ? a.det.bounds : a.bounds) + 10 * d;
    if (lane < 10) {
        const int k = lane >> 1;
        b[lane] = st == DS_OK ? (long long)((lane & 1) ? S.bd[k] : S.bn[k]) : 0;
    }
    if (lane == 0) {
        if (DETAIL) {
            a.det.status[d] = st;
            a.det.n_groups[d] = (unsigned short)ng;
            a.det.n_entities[d] = (unsigned short)nent;
            a.det.n_div_groups[d] = (unsigned short)ndiv;
        } else {
            a.status[d] = st;
            if (a.n_groups) a.n_groups[d] = (unsigned short)ng;
        }
    }
    __syncwarp();
}

// Main pass: every DAG of its size class (W=1: n <= 64; W=4: 64 < n <= 256;
// larger ones: k1_big),
// persistent warps striding over the batch, in 32-bit words. A DAG whose
// 32-bit pass overflows is queued for the 64-bit retry, and from there for
// the 128-bit one (k1_analyse_retry).
template <int W, bool DETAIL>
__global__ void __launch_bounds__(128) k1_analyse(const K1Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpState<W, u32>& S = reinterpret_cast<WarpState<W, u32>*>(smem_raw)[wib];
    const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
    const u32 nbase = a.node_off[0], ebase = a.edge_off[0];  // offsets are relative to element 0
    // a t_min that needs more than 32 bits sends every DAG to the wider tiers
    const bool narrow = ((a.plat.tmin.n | a.plat.tmin.d) >> 32) == 0;
    const PlatT<u32> P{a.plat.M, RatT<u32>{u32(a.plat.tmin.n), u32(a.plat.tmin.d)}, a.plat.minl};
    // W=1 takes DAGs dynamically (one atomic per DAG) so the per-DAG cost
    // spread does not leave a tail of idle SMs; W=4 only picks out the rare
    // big DAGs, statically.
    u32* const next = a.retry_count + 2;
    u64 d = W == 1 ? 0 : u64(blockIdx.x) * (blockDim.x >> 5) + wib;
#pragma unroll 1
    for (;; d += warps) {
        if (W == 1) {
            u32 t = 0;
            if (lane == 0) t = atomicAdd(next, 1u);
            d = __shfl_sync(FULL, t, 0);
        }
        if (d >= a.n_dags) break;
        const int n = int(a.node_off[d + 1] - a.node_off[d]);
        if (W > 1 && (n <= 64 || n > 256)) continue;  // k1_analyse<4>: 64 < n <= 256
        if (W == 1 && n > 64 && n <= DS_MAX_NODES) continue;  // the bigger kernels
        if (!narrow) {
            if (lane == 0) a.retry[atomicAdd(a.retry_count, 1u)] = u32(d);
            __syncwarp();
            continue;
        }
        run_one<W, u32, DETAIL>(S, lane, a, d, nbase, ebase, P, a.retry, a.retry_count);
    }
}

// k1_front: the W=1 main pass up to the division, 32-bit words.
template <bool UNUSED = false>  // a template so both K1 translation units may include it
__global__ void __launch_bounds__(128, 10) k1_front(const K1Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    WarpState<1, u32>& S = reinterpret_cast<WarpState<1, u32>*>(smem_raw)[threadIdx.x >> 5];
    const u32 nbase = a.node_off[0], ebase = a.edge_off[0];
    const bool narrow = ((a.plat.tmin.n | a.plat.tmin.d) >> 32) == 0;
    const PlatT<u32> P{a.plat.M, RatT<u32>{u32(a.plat.tmin.n), u32(a.plat.tmin.d)}, a.plat.minl};
    const bool proposed = a.mask & DS_M_PROPOSED;
    const u32 n_fb = a.fb_only ? a.retry_count[7] : 0u;  // written by k1_fast
#pragma unroll 1
    for (;;) {
        u32 t = 0;
        if (lane == 0) t = atomicAdd(a.retry_count + 2, 1u);
        t = __shfl_sync(FULL, t, 0);
        if (a.fb_only && t >= n_fb) break;
        const u64 d = a.fb_only ? a.h.fb[t] : t;
        if (d >= a.n_dags) break;
        if (!a.fb_only && a.h.skey && lane == 0) {
            a.h.skey[d] = kWalkKeyNone;  // not walked by k1_back_lane unless k1_mid keys it
        }
        const u32 n0 = a.node_off[d] - nbase, e0 = a.edge_off[d] - ebase;
        const int n = int(a.node_off[d + 1] - nbase - n0);
        if (n > 64 && n <= DS_MAX_NODES) continue;  // k1_analyse<4>
        int st = DS_EOVERFLOW, ng = 0, nent = 0, ndiv = 0;
        if (narrow) {
            st = analyse_dag<1, u32, false, true>(S, lane, n, a.load_num + n0, a.load_den ? a.load_den + n0 : nullptr,
                                                  a.edges + e0, a.edge_cnt ? int(a.edge_cnt[d]) : int(a.edge_off[d + 1] - ebase - e0), P, a.mask, ng,
                                                  DetailOut{}, nent, ndiv);
        }
        if (st == DS_EOVERFLOW) {
            if (lane == 0) {
                a.retry[atomicAdd(a.retry_count, 1u)] = u32(d);
                a.status[d] = kStRetried;
            }
            __syncwarp();
            continue;
        }
        const bool pending = st == DS_OK && proposed;
        int64_t* b = a.bounds + 10 * d;
        if (lane < 10 && !(pending && lane < 2)) {
            const int k = lane >> 1;
            b[lane] = st == DS_OK ? (long long)((lane & 1) ? S.bd[k] : S.bn[k]) : 0;
        }
        if (pending) {
#pragma unroll 1
            for (int v = lane; v < n; v += 32) {
                const u32 i = n0 + v;
                K1Node nd;
                nd.pred = S.pred[v][0];
                nd.ad = S.anc[v][0] | S.desc[v][0];  // k1_back only needs anc | desc
                nd.ln = S.ln[v];
                nd.ld = S.ld[v];
                nd.pad = 0;
                a.h.node[i] = nd;
                a.h.anc[i] = S.anc[v][0];
            }
        }
        if (lane == 0) {
            a.status[d] = pending ? kStMid : st;
            if (!pending && a.n_groups) a.n_groups[d] = 0;
        }
        __syncwarp();
    }
}

// k1_mid: ranks and division over k1_front's state.
template <bool UNUSED = false>
__global__ void __launch_bounds__(128) k1_mid(const K1Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    WarpState<1, u32>& S = reinterpret_cast<WarpState<1, u32>*>(smem_raw)[threadIdx.x >> 5];
    const u32 nbase = a.node_off[0];
    const PlatT<u32> P{a.plat.M, RatT<u32>{u32(a.plat.tmin.n), u32(a.plat.tmin.d)}, a.plat.minl};
    const u32 n_fb = a.fb_only ? a.retry_count[7] : 0u;
#pragma unroll 1
    for (;;) {
        u32 t = 0;
        if (lane == 0) t = atomicAdd(a.retry_count + 3, 1u);
        t = __shfl_sync(FULL, t, 0);
        if (a.fb_only && t >= n_fb) break;
        const u64 d = a.fb_only ? a.h.fb[t] : t;
        if (d >= a.n_dags) break;
        if (a.status[d] != kStMid) continue;
        const u32 n0 = a.node_off[d] - nbase;
        const int n = int(a.node_off[d + 1] - nbase - n0);
        bool integer = true;
#pragma unroll 1
        for (int v = lane; v < n; v += 32) {
            const u32 i = n0 + v;
            const K1Node& nd = a.h.node[i];
            S.pred[v][0] = nd.pred;
            S.anc[v][0] = a.h.anc[i];
            const RatT<u32> l{nd.ln, nd.ld};
            S.ln[v] = l.n;
            S.ld[v] = l.d;
            integer &= l.d == 1;
            S.mmax[v] = q_max_par(l, P);  // fits: k1_front computed it already
        }
        integer = __all_sync(FULL, integer);
        __syncwarp();
        const int n_joins = p_rank<1, u32>(S, lane, n, integer);
        if (n_joins < 0) {
            if (lane == 0) {
                a.retry[atomicAdd(a.retry_count, 1u)] = u32(d);
                a.status[d] = kStRetried;
            }
            __syncwarp();
            continue;
        }
        const int ndiv = p_division<1, u32, false>(S, lane, n, n_joins, P.M, DetailOut{});
#pragma unroll 1
        for (int v = lane; v < n; v += 32) {
            const u32 i = n0 + v;
            a.h.ro[i] = uint16_t(S.rank[v] | (S.order[v] << 8));
            if (v < ndiv) a.h.divg[i] = S.divg[v][0];
        }
        // shape key for the walk order: group count, then the member counts
        // (clipped to 3) of the first 10 division groups, group g in bits
        // 19-2g..18-2g — measured best of the keys tried (back 2.08 ms; with
        // only "which groups are multi-member" 2.11, member counts of 13
        // groups without the count 2.39, with the node count 2.20)
        const u32 cg = lane < ndiv ? u32(__popcll(S.divg[lane][0])) : 0u;
        const u32 cg2 = lane + 32 < ndiv ? u32(__popcll(S.divg[lane + 32][0])) : 0u;
        const u64 key = walk_key(lane, u32(ndiv), cg, cg2, false, a.key_mode);
        if (lane == 0) {
            a.h.ndiv[d] = uint16_t(ndiv);
            a.status[d] = kStPending;
            // within windows of kSortWindow consecutive DAGs (the window
            // index in the high bits), so a warp's walks stay near each other
            // in the hand-off and share L2 lines
            if (a.h.skey) a.h.skey[d] = key;
        }
        __syncwarp();
    }
}

// k1_back_lane: p_schedule with ONE LANE per DAG. The schedule is a
// sequential greedy over the executed groups (scheduler.cpp:214-359): in
// k1_back a warp walks it warp-uniformly, so 31 of 32 lanes replicate the
// scalar control flow (11 groups per C5 DAG, 70% singletons). Here every lane
// runs its own DAG's walk over the same k1_front/k1_mid state (read through
// L1 straight from the hand-off: the 32 DAGs of a warp are adjacent in it),
// so a warp instruction advances 32 DAGs. Same u32 words and the same
// helpers (exact rationals, overflow in-band as den 0); a DAG that overflows
// u32, or has more than kLaneMembers pending members in one group or more
// than kLaneSplits segmented nodes, goes to the retry tiers, which recompute
// it from scratch.
constexpr int kLaneMembers = 16;
constexpr int kLaneSplits = 8;
constexpr int kLaneRetry = -2;
constexpr int kLaneWarps = 4;
// Measured alternatives (ms, 1M C5 DAGs): this form 3.2-3.4; walking the groups
// in warp lock-step (__syncwarp per group) 3.64; the same walk as a state
// struct 3.66; staging the warp's 32 DAGs in shared memory 7.3 (residency
// fell to 12 warps/SM and the walk is latency bound). k1_back (warp per DAG)
// 4.40.

// The two hand-off layouts the walk reads (K1Node + ro + divg arrays, or the
// compact per-DAG K1Rec16 run): node v's load, anc|desc, preds; ro(i) =
// rank of node i | node at rank i << 8; division group g's member mask.
struct LaneWide {
    const K1Node* __restrict__ nodes;
    const uint16_t* __restrict__ r;
    const u64* __restrict__ g;
    __device__ __forceinline__ LaneWide(const K1Args& a, u32 n0) : nodes(a.h.node + n0), r(a.h.ro + n0), g(a.h.divg + n0) {}
    __device__ __forceinline__ RatT<u32> load(int v) const { return RatT<u32>{__ldg(&nodes[v].ln), __ldg(&nodes[v].ld)}; }
    __device__ __forceinline__ u64 ad(int v) const { return __ldg(&nodes[v].ad); }
    __device__ __forceinline__ u64 pred(int v) const { return __ldg(&nodes[v].pred); }
    __device__ __forceinline__ u32 ro(int i) const { return __ldg(r + i); }
    __device__ __forceinline__ u64 divg(int k) const { return __ldg(g + k); }
};
struct LaneCompact {
    const K1Rec16* __restrict__ rec;
    const u32* __restrict__ g;
    __device__ __forceinline__ LaneCompact(const K1Args& a, u32 n0, int n)
        : rec(reinterpret_cast<const K1Rec16*>(a.h.node + n0)), g(reinterpret_cast<const u32*>(rec + n)) {}
    __device__ __forceinline__ RatT<u32> load(int v) const { return RatT<u32>{__ldg(&rec[v].ln), 1u}; }
    __device__ __forceinline__ u64 ad(int v) const { return __ldg(&rec[v].ad); }
    __device__ __forceinline__ u64 pred(int v) const { return __ldg(&rec[v].pred); }
    __device__ __forceinline__ u32 ro(int i) const { return __ldg(&rec[i].ro); }
    __device__ __forceinline__ u64 divg(int k) const { return __ldg(g + k); }
};

template <int QB, class R>  // QB: bits per packed quota field, 8 (M <= 255) or 16 (M <= 65535)
__device__ __forceinline__ int schedule_lane(const R& H, const int n, const int ndiv, const PlatT<u32> P,
                                             RatT<u32>& bound, int& n_groups) {
    // residual loads of segmented nodes (scheduler.cpp:318-328), newest last
    int n_over = 0;
    int over_v[kLaneSplits];
    u32 over_n[kLaneSplits], over_d[kLaneSplits];
    auto load = [&](int v) -> RatT<u32> {
        for (int k = n_over - 1; k >= 0; --k) {
            if (over_v[k] == v) return RatT<u32>{over_n[k], over_d[k]};
        }
        return H.load(v);
    };
    bool ovf = false;
    const u64 V = n >= 64 ? ~0ull : ((1ull << n) - 1);
    RatT<u32> proposed{0, 1};
    u64 done = 0;
    int gidx = 0;
    u64 G_next = ndiv > 0 ? H.divg(0) : 0;  // one group ahead: off the dependent-load chain
#pragma unroll 1
    for (int g = 0; g < ndiv; ++g) {
        const u64 G = G_next;
        if (g + 1 < ndiv) G_next = H.divg(g + 1);
        const u64 org = G & ~done;
        if (!org) continue;  // fully absorbed by earlier launches
        RatT<u32> R{0, 1};
        int used = 0;
        u64 conc = 0;  // union of the members' concurrent sets (+ themselves)
        if (!(org & (org - 1))) {
            // one pending member: m = min(m^max, M), no shed/fill
            const int v = __ffsll(org) - 1;
            const RatT<u32> l = load(v);
            int cp = q_max_par(l, P);
            if (cp < 0) {
                ovf = true;
                cp = 1;
            }
            cp = min(cp, P.M);
            R = q_exec(l, cp, P);
            ovf |= R.d == 0;
            used = cp;
            conc = ~H.ad(v);
        } else {
            // apportion (scheduler.cpp:35-95) over the pending loads. Member k's
            // quota (<= M) lives in an 8-bit field (M <= 255) or a 16-bit
            // field (M <= 65535) of the packed words mq (registers, no local
            // memory); cap and quota remainder are recomputed where needed.
            if (__popcll(org) > kLaneMembers || P.M >= (1 << QB)) return kLaneRetry;
            u64 mq[QB == 8 ? 2 : 4] = {};
            constexpr int lw = QB == 8 ? 3 : 4;  // log2 bits per field
            constexpr int lper = 6 - lw;         // log2 fields per word
            constexpr u64 fmask = (1ull << QB) - 1;
            auto get = [&](int k) {
                return int((mq[k >> lper] >> ((k & ((1 << lper) - 1)) << lw)) & fmask);
            };
            auto put = [&](int k, int m) {
                const int sh = (k & ((1 << lper) - 1)) << lw;
                mq[k >> lper] = (mq[k >> lper] & ~(fmask << sh)) | (u64(m) << sh);
            };
            RatT<u32> Wt{0, 1};
#pragma unroll 1
            for (u64 b = org; b; b &= b - 1) Wt = q_add(Wt, load(__ffsll(b) - 1));
            if (Wt.d == 0 || Wt.n == 0) return DS_EOVERFLOW;
            auto cap_of = [&](const RatT<u32>& l) {
                int cp = q_max_par(l, P);
                if (cp < 0) {
                    ovf = true;
                    cp = 1;
                }
                return min(cp, P.M);
            };
            // quota = l*M/W = (l.n*M*W.d) / (l.d*W.n): floor and remainder
            auto quota = [&](const RatT<u32>& l, u32& qn, u32& qd) {
                qn = mulc(mulc(l.n, u32(P.M), ovf), Wt.d, ovf);
                qd = mulc(l.d, Wt.n, ovf);
                return qd ? qn / qd : 0u;
            };
            int tot = 0, capsum = 0, nm = 0;
#pragma unroll 1
            for (u64 b = org; b; b &= b - 1, ++nm) {
                const RatT<u32> l = load(__ffsll(b) - 1);
                const int cp = cap_of(l);
                u32 qn, qd;
                const u32 fl = quota(l, qn, qd);
                if (qd == 0) return DS_EOVERFLOW;
                const long long flc = fl > 0x7fffffffu ? 0x7fffffffll : (long long)fl;
                const int base = int(max(1ll, min(flc, (long long)cp)));
                put(nm, base);
                tot += base;
                capsum += cp;
            }
            const int target = min(P.M, capsum);
#pragma unroll 1
            while (tot > P.M || tot < target) {
                const bool shed = tot > P.M;
                Pick<u32> c{{0, 1}, {0, 1}, -1};
                int ck = -1, k = 0;
#pragma unroll 1
                for (u64 b = org; b; b &= b - 1, ++k) {
                    const int v = __ffsll(b) - 1;
                    const int m = get(k);
                    const RatT<u32> l = load(v);
                    if (shed ? m <= 1 : m >= cap_of(l)) continue;
                    RatT<u32> k2{0, 1};
                    if (!shed) {
                        u32 qn, qd;
                        const u32 fl = quota(l, qn, qd);
                        k2 = RatT<u32>{qn - fl * qd, qd};
                    }
                    const Pick<u32> x{q_exec_raw(l, shed ? m - 1 : m, P), k2, v};
                    ovf |= x.k1.d == 0;
                    if (pick_better<u32>(x, c, shed)) {
                        c = x;
                        ck = k;
                    }
                }
                if (ck < 0) return DS_EINVARIANT;
                const int step = shed ? -1 : 1;
                put(ck, get(ck) + step);
                tot += step;
            }
            // members: exec, response = first strict max
            bool first = true;
            int k = 0;
#pragma unroll 1
            for (u64 b = org; b; b &= b - 1, ++k) {
                const int v = __ffsll(b) - 1;
                const int m = get(k);
                const RatT<u32> e = q_exec(load(v), m, P);
                ovf |= e.d == 0;
                if (first || q_cmp(e, R) > 0) {
                    R = e;
                    first = false;
                }
                used += m;
                conc |= ~H.ad(v);
            }
        }
        const int spare0 = P.M - used;
        // candidates (scheduler.cpp:253-280): sources of the pool that are
        // released, launched in rank order (:286-330)
        const u64 pool = V & conc & ~G;
        const u64 avail = pool & ~done;
        u64 whole = 0;
        if (avail && spare0 >= 1) {
            u64 rm = 0;
            // two candidates per step: their loads are independent
#pragma unroll 1
            for (u64 b = avail; b;) {
                const int c0 = __ffsll(b) - 1;
                b &= b - 1;
                const int c1 = b ? __ffsll(b) - 1 : -1;
                b &= b - 1;
                const u64 p0 = H.pred(c0);
                const u64 p1 = c1 >= 0 ? H.pred(c1) : ~0ull;
                const u32 r0 = H.ro(c0);
                const u32 r1 = c1 >= 0 ? H.ro(c1) : 0;
                if (!(p0 & pool) && !(p0 & ~done)) rm |= 1ull << (r0 & 0xff);
                if (c1 >= 0 && !(p1 & pool) && !(p1 & ~done)) rm |= 1ull << (r1 & 0xff);
            }
            int spare = spare0;
#pragma unroll 1
            for (; rm && spare >= 1; rm &= rm - 1) {
                const int c = int(H.ro(__ffsll(rm) - 1) >> 8);
                const RatT<u32> l = load(c);
                int mp = q_max_par(l, P);
                if (mp < 0) {
                    ovf = true;
                    mp = 1;
                }
                const int mc = min(mp, spare);
                const RatT<u32> dur = q_exec(l, mc, P);
                ovf |= dur.d == 0;
                spare -= mc;
                if (q_cmp(dur, R) <= 0) {
                    whole |= 1ull << c;
                } else {  // split: the residual replaces the origin
                    const RatT<u32> pl = n_mul_int(R, u32(mc));
                    const RatT<u32> rl = n_sub(l, pl);
                    ovf |= pl.d == 0 || rl.d == 0;
                    if (n_over == kLaneSplits) return kLaneRetry;
                    over_v[n_over] = c;
                    over_n[n_over] = rl.n;
                    over_d[n_over] = rl.d;
                    ++n_over;
                    break;
                }
            }
        }
        done |= org | whole;
        proposed = q_add(proposed, R);
        ovf |= proposed.d == 0;
        ++gidx;
    }
    if (ovf) return DS_EOVERFLOW;
    if (done != V) return DS_EINVARIANT;  // "scheduling finished with unplaced kernels"
    bound = proposed;
    n_groups = gidx;
    return DS_OK;
}

#ifndef DS_LANE_MIN_BLOCKS
#define DS_LANE_MIN_BLOCKS 9  // 56 registers: 3.02 ms; 64 regs 3.09, 48 regs 3.07, 40 regs 3.09 (1M C5 DAGs)
#endif
template <bool UNUSED = false, int QB = 8>
__global__ void __launch_bounds__(32 * kLaneWarps, DS_LANE_MIN_BLOCKS) k1_back_lane(const K1Args a) {
    const int lane = threadIdx.x & 31;
    const u32 nbase = a.node_off[0];
    const PlatT<u32> P{a.plat.M, RatT<u32>{u32(a.plat.tmin.n), u32(a.plat.tmin.d)}, a.plat.minl};
    // Task order. Default: 32 consecutive walk-order positions per task. With
    // wcnt (heavy-first): three phases of per-window task slots (128 per
    // window) — every window's wide DAGs (n > 32, the longest walks), then
    // its compact DAGs with many division groups, then the rest — so the last
    // wave of tasks holds short walks and the kernel's tail shrinks; windows
    // stay in order within a phase (L2 locality), and empty slots are skipped
    // after one counter read.
    // Only the last ~two waves of windows are phased (the tail is the last
    // wave); earlier windows go in plain window order, which keeps a warp's
    // hand-off reads inside a compact address range (L2 hits).
    const u64 nwin = (a.n_dags + kSortWindow - 1) / kSortWindow;
    const u64 wave = u64(gridDim.x) * (blockDim.x >> 5) * 32;  // DAGs one wave of warp tasks covers
    const u64 w0 = a.n_dags > 2 * wave ? (a.n_dags - 2 * wave) / kSortWindow : 0;  // first phased window
    const u64 plain = w0 * (kSortWindow / 32), slots = (nwin - w0) * (kSortWindow / 32);
#pragma unroll 1
    for (;;) {
        u32 t = 0;
        if (lane == 0) t = atomicAdd(a.retry_count + 5, a.h.wcnt ? 1u : 32u);
        t = __shfl_sync(FULL, t, 0);
        u64 q;
        if (a.h.wcnt && t < plain) {
            q = u64(t) * 32 + lane;  // windows [0, w0): walk order as sorted
        } else if (a.h.wcnt) {
            const u64 tp = t - plain;
            if (tp >= 3 * slots) break;
            const int cls = 2 - int(tp / slots);  // 2 wide, 1 heavy compact, 0 light compact
            const u64 sl = tp % slots, w = w0 + sl / (kSortWindow / 32), k = sl % (kSortWindow / 32);
            const u32* c = a.h.wcnt + 3 * w;
            const u32 cnt = c[cls], start = cls == 0 ? 0u : cls == 1 ? c[0] : c[0] + c[1];
            if (32 * k >= cnt) continue;
            if (32 * k + lane >= cnt) continue;
            q = w * kSortWindow + start + 32 * k + lane;
        } else {
            if (t >= a.n_dags) break;
            q = u64(t) + lane;
            if (q >= a.n_dags) continue;
        }
        const u64 d = a.perm ? u64(a.perm[q]) : q;
        if (a.status[d] != kStPending) continue;
        const u32 n0 = a.node_off[d] - nbase;
        const int n = int(a.node_off[d + 1] - nbase - n0);
        RatT<u32> bound{0, 0};
        int ng = 0;
        const uint16_t nd = a.h.ndiv[d];
        const int st = (nd & kNdivCompact)
                           ? schedule_lane<QB>(LaneCompact(a, n0, n), n, nd & ~kNdivCompact, P, bound, ng)
                           : schedule_lane<QB>(LaneWide(a, n0), n, nd, P, bound, ng);
        if (st == DS_EOVERFLOW || st == kLaneRetry) {  // recomputed from scratch in wider words
            a.retry[atomicAdd(a.retry_count, 1u)] = u32(d);
            a.status[d] = kStRetried;
            continue;
        }
        int64_t* b = a.bounds + 10 * d;
        if (st == DS_OK) {
            b[0] = (long long)bound.n;
            b[1] = (long long)bound.d;
        } else {
            for (int k = 0; k < 10; ++k) b[k] = 0;
        }
        a.status[d] = st;
        if (a.n_groups) a.n_groups[d] = (unsigned short)(st == DS_OK ? ng : 0);
    }
}

// Retry passes over the DAGs queued by the narrower tier: T = u64 reads
// retry/retry_count and queues its own overflows in retry2; T = u128 is final.
template <bool DETAIL, class T>
__global__ void __launch_bounds__(32) k1_analyse_retry(const K1Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    WarpState<4, T>& S = *reinterpret_cast<WarpState<4, T>*>(smem_raw);
    const PlatT<T> P{a.plat.M, RatT<T>{T(a.plat.tmin.n), T(a.plat.tmin.d)}, a.plat.minl};
    const u32 nbase = a.node_off[0], ebase = a.edge_off[0];
    constexpr bool wide = sizeof(T) == 16;
    const u32* list = wide ? a.retry2 : a.retry;
    const u32 count = *(wide ? a.retry2_count : a.retry_count);
#pragma unroll 1
    for (u32 i = blockIdx.x; i < count; i += gridDim.x) {
        run_one<4, T, DETAIL>(S, lane, a, list[i], nbase, ebase, P, wide ? nullptr : a.retry2,
                              wide ? nullptr : a.retry2_count);
    }
}

}  // namespace ds

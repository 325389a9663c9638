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
// v % 32 (2W nodes per lane); the inherently sequential parts of the greedy
// (group loop, apportion shed/fill, launch loop) run warp-uniformly over
// masks, so there is no divergence and no shuffle traffic in them.
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

template <int W>
struct WarpState {
    static constexpr int N = 64 * W;
    u64 pred[N][W], succ[N][W], anc[N][W], desc[N][W];
    u64 divg[N][W];              // division groups, in order
    u64 ln[N], ld[N];            // original load
    u64 pn[N], pd[N];            // pending load (residual after a split)
    u64 xn[N], xd[N];            // W^anc, later per-member exec
    u64 rn[N], rd[N];            // apportion remainder (unreduced)
    u64 cn[N], cd[N];            // critical-path prefix (lower bound)
    int mmax[N];                 // max_parallelism(original load)
    int mq[N];                   // apportioned parallelism
    int cap[N];                  // min(max_parallelism(pending load), M)
    short rank[N];               // position in (W^anc desc, id asc)
    short order[N];              // node at rank r
    short jorder[N];             // joins in (W^anc asc, id asc)
    short done[N];               // executed group that completed the origin, -1 pending
    unsigned short gen[N];       // split generation counter
    unsigned char level[N];      // 1 + longest predecessor chain (hop count)
    unsigned char ppart[N];      // pending entity part (0 whole, 2 residual)
    u64 rmask[W];                // rank-space scratch
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
};

template <int W>
__device__ __forceinline__ Mask<W> load_mask(const u64 (&m)[W]) {
    Mask<W> r;
#pragma unroll
    for (int k = 0; k < W; ++k) r.w[k] = m[k];
    return r;
}

// Uniform mask from a per-node predicate evaluated by the owning lanes.
template <int W, class Pred>
__device__ __forceinline__ Mask<W> ballot_nodes(int lane, Pred pred) {
    Mask<W> r;
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const u32 lo = __ballot_sync(FULL, pred(k * 64 + lane));
        const u32 hi = __ballot_sync(FULL, pred(k * 64 + 32 + lane));
        r.w[k] = u64(lo) | (u64(hi) << 32);
    }
    return r;
}

// Iterate the set bits of a uniform mask in ascending node order.
template <int W, class F>
__device__ __forceinline__ void for_bits(const Mask<W>& m, F f) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
        for (u64 x = m.w[k]; x; x &= x - 1) f(k * 64 + __ffsll(x) - 1);
    }
}

struct DetailOut {
    ds_entity_rec* ent;  // this DAG's entity slots
    ds_group_rec* grp;   // this DAG's group slots
    short* node_block;
    short* node_div_group;
};

// Analyse DAG `d`. All lanes of the warp call this with identical arguments.
// Returns the DS_* status; writes bounds (and detail records when DETAIL).
template <int W, bool DETAIL>
__device__ int analyse_dag(WarpState<W>& S, const int lane, const int n, const u64* __restrict__ lnum,
                           const u64* __restrict__ lden, const u32* __restrict__ edges, const int n_edges,
                           const Plat P, const u32 mask, Rat (&bound)[DS_N_BOUNDS], int& n_groups_out,
                           DetailOut det, int& n_ent_out, int& n_div_out) {
    constexpr int N = WarpState<W>::N;
    bool ovf = false;
    n_groups_out = 0;
    n_ent_out = 0;
    n_div_out = 0;
    if (n <= 0) return DS_E_EMPTY;
    if (n > N) return DS_ETOOBIG;

    // ---------------------------------------------------------------- loads
    // dag.cpp:35-41 (load >= min_load; min_load = t_min on this path)
    bool bad_load = false, bad_arg = false, frac = false;
    for (int v = lane; v < N; v += 32) {
        if (v < n) {
            long long a = (long long)lnum[v];
            long long b = lden ? (long long)lden[v] : 1;
            if (b == 0) bad_arg = true;
            if (b < 0) {
                a = -a;
                b = -b;
            }
            Rat l = a > 0 && b > 0 ? rat_reduce(u64(a), u64(b)) : Rat{0, 1};
            if (a <= 0 || rat_cmp(l, P.tmin) < 0) bad_load = true;
            frac |= l.d != 1;
            S.ln[v] = l.n;
            S.ld[v] = l.d;
            S.pn[v] = l.n;
            S.pd[v] = l.d;
            S.mmax[v] = (a > 0 && b > 0) ? max_par(l, P) : 1;
            S.done[v] = -1;
            S.gen[v] = 0;
            S.ppart[v] = 0;
            S.level[v] = 0;
        }
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
    const bool integer_loads = !__any_sync(FULL, frac);
    __syncwarp();

    // ---------------------------------------------------------------- edges
    // dag.cpp:48-67: checked in sorted (from, to) order; first failure wins.
    u32 first_bad = 0xffffffffu;
    int bad_kind = 0;
    for (int e = lane; e < n_edges; e += 32) {
        const u32 w = edges[e];
        const int u = int(w >> 16), v = int(w & 0xffffu);
        if (u >= n || v >= n || u == v) {
            if (w < first_bad) {
                first_bad = w;
                bad_kind = (u >= n || v >= n) ? DS_E_EDGE : DS_E_SELFLOOP;
            }
        } else {
            atomicOr(&S.succ[u][v >> 6], 1ull << (v & 63));
            atomicOr(&S.pred[v][u >> 6], 1ull << (u & 63));
        }
    }
    {
        const u32 m = __reduce_min_sync(FULL, first_bad);
        if (m != 0xffffffffu) {
            const u32 who = __ballot_sync(FULL, first_bad == m);
            return __shfl_sync(FULL, bad_kind, __ffs(who) - 1);
        }
    }
    __syncwarp();

    Mask<W> V;
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int lo = k * 64, hi = lo + 64;
        V.w[k] = n >= hi ? ~0ull : (n <= lo ? 0ull : ((1ull << (n - lo)) - 1));
    }

    // ------------------------------------------- closure (Kahn, level-synchronous)
    // dag.cpp:69-124. Round r makes ready every node whose predecessors are
    // all processed; a node's round is 1 + the longest predecessor chain (the
    // hop count graham_para needs). No progress with nodes left = cycle.
    const bool want_lower = mask & DS_M_LOWER;
    if (want_lower) {
        for (int v = lane; v < n; v += 32) {
            Rat w = exec_time(Rat{S.ln[v], S.ld[v]}, min(S.mmax[v], P.M), P, ovf);
            S.cn[v] = w.n;  // weight; replaced by the path prefix below
            S.cd[v] = w.d;
        }
    }
    Mask<W> done_m;
    done_m.clear();
    int rounds = 0;
    for (;;) {
        const Mask<W> R = ballot_nodes<W>(lane, [&](int v) {
            if (v >= n || done_m.test(v)) return false;
            bool ok = true;
#pragma unroll
            for (int k = 0; k < W; ++k) ok &= (S.pred[v][k] & ~done_m.w[k]) == 0;
            return ok;
        });
        if (!R.any()) break;
        ++rounds;
        for (int v = lane; v < N; v += 32) {
            if (!R.test(v)) continue;
            u64 a[W];
#pragma unroll
            for (int k = 0; k < W; ++k) a[k] = 0;
            Rat best{0, 1};
            const Mask<W> pm = load_mask<W>(S.pred[v]);
            for_bits<W>(pm, [&](int p) {
#pragma unroll
                for (int k = 0; k < W; ++k) a[k] |= S.anc[p][k];
                a[p >> 6] |= 1ull << (p & 63);
                if (want_lower) best = rat_max(best, Rat{S.cn[p], S.cd[p]});
            });
#pragma unroll
            for (int k = 0; k < W; ++k) S.anc[v][k] = a[k];
            S.level[v] = (unsigned char)min(rounds, 255);
            if (want_lower) {
                Rat c = rat_add(best, Rat{S.cn[v], S.cd[v]}, ovf);
                S.cn[v] = c.n;
                S.cd[v] = c.d;
            }
        }
#pragma unroll
        for (int k = 0; k < W; ++k) done_m.w[k] |= R.w[k];
        __syncwarp();
    }
    {
        bool all = true;
#pragma unroll
        for (int k = 0; k < W; ++k) all &= done_m.w[k] == V.w[k];
        if (!all) return DS_E_CYCLE;
    }
    // dag.cpp:97-108: exactly one source and one sink
    {
        const Mask<W> src = ballot_nodes<W>(lane, [&](int v) {
            if (v >= n) return false;
            u64 a = 0;
#pragma unroll
            for (int k = 0; k < W; ++k) a |= S.pred[v][k];
            return a == 0;
        });
        if (src.popc() != 1) return DS_E_SOURCES;
        const Mask<W> snk = ballot_nodes<W>(lane, [&](int v) {
            if (v >= n) return false;
            u64 a = 0;
#pragma unroll
            for (int k = 0; k < W; ++k) a |= S.succ[v][k];
            return a == 0;
        });
        if (snk.popc() != 1) return DS_E_SINKS;
    }
    // descendants: reverse rounds over successors
    done_m.clear();
    for (;;) {
        const Mask<W> R = ballot_nodes<W>(lane, [&](int v) {
            if (v >= n || done_m.test(v)) return false;
            bool ok = true;
#pragma unroll
            for (int k = 0; k < W; ++k) ok &= (S.succ[v][k] & ~done_m.w[k]) == 0;
            return ok;
        });
        if (!R.any()) break;
        for (int v = lane; v < N; v += 32) {
            if (!R.test(v)) continue;
            u64 a[W];
#pragma unroll
            for (int k = 0; k < W; ++k) a[k] = 0;
            const Mask<W> sm = load_mask<W>(S.succ[v]);
            for_bits<W>(sm, [&](int s) {
#pragma unroll
                for (int k = 0; k < W; ++k) a[k] |= S.desc[s][k];
                a[s >> 6] |= 1ull << (s & 63);
            });
#pragma unroll
            for (int k = 0; k < W; ++k) S.desc[v][k] = a[k];
        }
#pragma unroll
        for (int k = 0; k < W; ++k) done_m.w[k] |= R.w[k];
        __syncwarp();
    }

    // ---------------------------------------------------------------- bounds
    // analysis.cpp:40-81 (node-parallel sums; canonical rationals)
    if (mask & (DS_M_GREEDY | DS_M_GREEDY_UNAWARE | DS_M_GRAHAM_PARA | DS_M_LOWER)) {
        Rat g{0, 1}, gu{0, 1}, tot{0, 1};
        u64 units = 0;
        for (int v = lane; v < n; v += 32) {
            const Rat l{S.ln[v], S.ld[v]};
            if (mask & DS_M_GREEDY) g = rat_add(g, exec_time(l, min(S.mmax[v], P.M), P, ovf), ovf);
            if (mask & DS_M_GREEDY_UNAWARE) gu = rat_add(gu, exec_time(l, S.mmax[v], P, ovf), ovf);
            if (mask & DS_M_GRAHAM_PARA) units += rat_ceil(rat_div(l, P.tmin, ovf));
            if (mask & DS_M_LOWER) tot = rat_add(tot, l, ovf);
        }
        if (mask & DS_M_GREEDY) bound[DS_BOUND_GREEDY] = warp_sum(g, ovf);
        if (mask & DS_M_GREEDY_UNAWARE) bound[DS_BOUND_GREEDY_UNAWARE] = warp_sum(gu, ovf);
        if (mask & DS_M_GRAHAM_PARA) {
#pragma unroll
            for (int o = 16; o; o >>= 1) units += __shfl_xor_sync(FULL, units, o);
            // chain = (longest hop path) * t_min; bound = chain + (work - chain) / M
            const Rat work = rat_mul_int(P.tmin, units, ovf);
            const Rat chain = rat_mul_int(P.tmin, u64(rounds), ovf);
            bound[DS_BOUND_GRAHAM_PARA] =
                rat_add(chain, rat_div_int(rat_sub(work, chain, ovf), u64(P.M), ovf), ovf);
        }
        if (mask & DS_M_LOWER) {
            tot = warp_sum(tot, ovf);
            Rat cp{0, 1};
            for (int v = lane; v < n; v += 32) cp = rat_max(cp, Rat{S.cn[v], S.cd[v]});
            cp = warp_max(cp);
            bound[DS_BOUND_LOWER] = rat_max(rat_div_int(tot, u64(P.M), ovf), cp);
        }
    }

    const bool need_sched = (mask & DS_M_PROPOSED) || DETAIL;
    if (!need_sched) return __any_sync(FULL, ovf) ? DS_EOVERFLOW : DS_OK;

    // ----------------------------------------------------------- W^anc, ranks
    // dag.cpp:126-135 W^anc = load + sum of ancestors' loads
    for (int v = lane; v < n; v += 32) {
        const Mask<W> am = load_mask<W>(S.anc[v]);
        if (integer_loads) {
            u64 s = S.ln[v];
            for_bits<W>(am, [&](int u) { s = addc(s, S.ln[u], ovf); });
            S.xn[v] = s;
            S.xd[v] = 1;
        } else {
            Rat s{S.ln[v], S.ld[v]};
            for_bits<W>(am, [&](int u) { s = rat_add(s, Rat{S.ln[u], S.ld[u]}, ovf); });
            S.xn[v] = s.n;
            S.xd[v] = s.d;
        }
    }
    __syncwarp();
    // rank in (W^anc desc, id asc) — heads (division.cpp:88-93) and
    // candidates (scheduler.cpp:275-280); join order (W^anc asc, id asc,
    // dag.cpp:218-230) among joins.
    int n_joins = 0;
    {
        const Mask<W> J = ballot_nodes<W>(lane, [&](int v) {
            if (v >= n) return false;
            int c = 0;
#pragma unroll
            for (int k = 0; k < W; ++k) c += __popcll(S.pred[v][k]);
            return c >= 2;
        });
        n_joins = J.popc();
        for (int v = lane; v < n; v += 32) {
            const Rat wv{S.xn[v], S.xd[v]};
            int r = 0, jr = 0;
            const bool isj = J.test(v);
            for (int u = 0; u < n; ++u) {
                const Rat wu{S.xn[u], S.xd[u]};
                const int c = integer_loads ? (wu.n < wv.n ? -1 : (wu.n > wv.n ? 1 : 0)) : rat_cmp(wu, wv);
                r += (c > 0) || (c == 0 && u < v);
                if (isj) jr += J.test(u) && ((c < 0) || (c == 0 && u < v));
            }
            S.rank[v] = short(r);
            S.order[r] = short(v);
            if (isj) S.jorder[jr] = short(v);
        }
    }
    __syncwarp();

    // -------------------------------------------------------------- division
    // division.cpp:10-30 blocks in join order + residual; :67-126 groups.
    int n_div = 0;
    Mask<W> assigned;
    assigned.clear();
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
            for (int v = lane; v < n; v += 32) {
                if (B.test(v)) det.node_block[v] = short(b);
            }
        }
        Mask<W> grouped;
        grouped.clear();
        for (;;) {
            // heads: ungrouped members whose in-block predecessor is grouped or absent
            const Mask<W> H = ballot_nodes<W>(lane, [&](int v) {
                if (v >= n || !B.test(v) || grouped.test(v)) return false;
                bool ok = true;
#pragma unroll
                for (int k = 0; k < W; ++k) ok &= (S.pred[v][k] & B.w[k] & ~grouped.w[k]) == 0;
                return ok;
            });
            if (!H.any()) break;
            Mask<W> sel = H;
            if (H.popc() > P.M) {  // keep the top-M by rank
#pragma unroll
                for (int k = 0; k < W; ++k) S.rmask[k] = 0;
                __syncwarp();
                for (int v = lane; v < n; v += 32) {
                    if (H.test(v)) atomicOr(&S.rmask[S.rank[v] >> 6], 1ull << (S.rank[v] & 63));
                }
                __syncwarp();
                sel = ballot_nodes<W>(lane, [&](int v) {
                    if (v >= n || !H.test(v)) return false;
                    const int r = S.rank[v];
                    int below = 0;
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        const u64 w = S.rmask[k];
                        if (k * 64 + 64 <= r) below += __popcll(w);
                        else if (k * 64 < r) below += __popcll(w & ((1ull << (r - k * 64)) - 1));
                    }
                    return below < P.M;
                });
                __syncwarp();
            }
            // Rule 2: any selected head with m^max >= M -> the max-m^max head alone
            int mx = 0;
            for (int v = lane; v < n; v += 32) {
                if (sel.test(v)) mx = max(mx, S.mmax[v]);
            }
            mx = __reduce_max_sync(FULL, mx);
            if (mx >= P.M) {
                const Mask<W> top = ballot_nodes<W>(lane, [&](int v) {
                    return v < n && sel.test(v) && S.mmax[v] == mx;
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
                for (int v = lane; v < n; v += 32) {
                    if (sel.test(v)) det.node_div_group[v] = short(n_div);
                }
            }
            ++n_div;
        }
    }
    __syncwarp();
    n_div_out = n_div;

    // --------------------------------------------------------------- schedule
    // scheduler.cpp:214-359, one executed group per non-absorbed division group
    Rat proposed{0, 1};
    int gidx = 0, n_ent = 0;
    Mask<W> done_mask;
    done_mask.clear();
    for (int g = 0; g < n_div; ++g) {
        const Mask<W> G = load_mask<W>(S.divg[g]);
        Mask<W> org;
#pragma unroll
        for (int k = 0; k < W; ++k) org.w[k] = G.w[k] & ~done_mask.w[k];
        if (!org.any()) continue;  // fully absorbed by earlier launches

        // -- apportion (scheduler.cpp:35-95) over pending loads
        Rat Wt{0, 1};
        for_bits<W>(org, [&](int v) { Wt = rat_add(Wt, Rat{S.pn[v], S.pd[v]}, ovf); });
        int tot = 0, capsum = 0;
        for (int v = lane; v < n; v += 32) {
            if (!org.test(v)) continue;
            const Rat l{S.pn[v], S.pd[v]};
            const int cp = min(max_par(l, P), P.M);
            // quota = l*M/W = (l.n*M*W.d) / (l.d*W.n)
            unsigned __int128 qn = (unsigned __int128)mulc(l.n, u64(P.M), ovf) * Wt.d;
            unsigned __int128 qd = (unsigned __int128)l.d * Wt.n;
            u64 fl, rem_n, rem_d;
            if (((qn | qd) >> 64) == 0) {
                const u64 a = u64(qn), c = u64(qd);
                fl = div64(a, c);
                rem_n = a - fl * c;
                rem_d = c;
            } else {
                const unsigned __int128 f = qn / qd;
                const unsigned __int128 r = qn - f * qd;
                if ((f >> 63) || (r >> 64) || (qd >> 64)) ovf = true;
                fl = u64(f);
                rem_n = u64(r);
                rem_d = u64(qd);
            }
            const long long base = max(1ll, min((long long)min(fl, u64(0x7fffffffffffll)), (long long)cp));
            S.mq[v] = int(base);
            S.cap[v] = cp;
            S.rn[v] = rem_n;
            S.rd[v] = rem_d;
            tot += int(base);
            capsum += cp;
        }
        tot = __reduce_add_sync(FULL, tot);
        capsum = __reduce_add_sync(FULL, capsum);
        __syncwarp();
        while (tot > P.M) {  // shed: smallest slowdown, first index wins ties
            int pick = -1;
            Rat best{0, 1};
            for_bits<W>(org, [&](int v) {
                const int m = S.mq[v];
                if (m <= 1) return;
                const Rat s = exec_raw(Rat{S.pn[v], S.pd[v]}, m - 1, P, ovf);
                if (pick < 0 || rat_cmp(s, best) < 0) {
                    pick = v;
                    best = s;
                }
            });
            if (pick < 0) return DS_EINVARIANT;
            if (lane == 0) S.mq[pick] -= 1;
            __syncwarp();
            --tot;
        }
        const int target = min(P.M, capsum);
        while (tot < target) {  // fill: largest exec, then larger remainder, then first index
            int pick = -1;
            Rat be{0, 1}, br{0, 1};
            for_bits<W>(org, [&](int v) {
                const int m = S.mq[v];
                if (m >= S.cap[v]) return;
                const Rat cur = exec_raw(Rat{S.pn[v], S.pd[v]}, m, P, ovf);
                const Rat rm{S.rn[v], S.rd[v]};
                int c = 1;
                if (pick >= 0) {
                    c = rat_cmp(cur, be);
                    if (c == 0) c = rat_cmp(rm, br);
                }
                if (c > 0) {
                    pick = v;
                    be = cur;
                    br = rm;
                }
            });
            if (pick < 0) return DS_EINVARIANT;
            if (lane == 0) S.mq[pick] += 1;
            __syncwarp();
            ++tot;
        }

        // -- members: exec, response (first strict max), bottleneck
        for (int v = lane; v < n; v += 32) {
            if (!org.test(v)) continue;
            const Rat e = exec_time(Rat{S.pn[v], S.pd[v]}, S.mq[v], P, ovf);
            S.xn[v] = e.n;
            S.xd[v] = e.d;
        }
        __syncwarp();
        Rat R{0, 1};
        int bott = -1, used = 0, n_mem = 0, bott_pos = 0;
        for_bits<W>(org, [&](int v) {
            const Rat e{S.xn[v], S.xd[v]};
            if (bott < 0 || rat_cmp(e, R) > 0) {
                R = e;
                bott = v;
                bott_pos = n_mem;
            }
            used += S.mq[v];
            ++n_mem;
        });
        const int spare0 = P.M - used;

        // -- candidates (scheduler.cpp:253-280). Concurrency is symmetric, so
        // c is in the pool iff some pending member is concurrent with c.
        const Mask<W> pool = ballot_nodes<W>(lane, [&](int c) {
            if (c >= n || G.test(c)) return false;
            u64 hit = 0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                u64 con = V.w[k] & ~(S.anc[c][k] | S.desc[c][k]);
                if ((c >> 6) == k) con &= ~(1ull << (c & 63));
                hit |= con & org.w[k];
            }
            return hit != 0;
        });
        const Mask<W> cands = ballot_nodes<W>(lane, [&](int c) {
            if (c >= n || !pool.test(c) || done_mask.test(c)) return false;
            bool ok = true;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                ok &= (S.pred[c][k] & pool.w[k]) == 0;       // source of the pool
                ok &= (S.pred[c][k] & ~done_mask.w[k]) == 0; // released (preds done earlier)
            }
            return ok;
        });

        // -- launches in rank order (scheduler.cpp:286-330)
        Mask<W> whole;
        whole.clear();
        int spare = spare0, n_launch = 0;
        const int first_ent = n_ent;
        if (cands.any() && spare >= 1) {
#pragma unroll
            for (int k = 0; k < W; ++k) S.rmask[k] = 0;
            __syncwarp();
            for (int v = lane; v < n; v += 32) {
                if (cands.test(v)) atomicOr(&S.rmask[S.rank[v] >> 6], 1ull << (S.rank[v] & 63));
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
                const Rat l{S.pn[c], S.pd[c]};
                const int mc = min(max_par(l, P), spare);
                const Rat dur = exec_time(l, mc, P, ovf);
                if (rat_cmp(dur, R) <= 0) {
                    if (DETAIL && lane == 0) {
                        ds_entity_rec& e = det.ent[n_ent];
                        e.origin = (unsigned short)c;
                        e.generation = S.gen[c];
                        e.part = S.ppart[c];
                        e.launched = 1;
                        e.group = (unsigned short)gidx;
                        e.parallelism = mc;
                        e.load_num = (long long)l.n;
                        e.load_den = (long long)l.d;
                        e.exec_num = (long long)dur.n;
                        e.exec_den = (long long)dur.d;
                        e.res_num = 0;
                        e.res_den = 0;
                    }
                    whole.set(c);
                    if (lane == 0) S.done[c] = short(gidx);
                    spare -= mc;
                } else {
                    const Rat pl = rat_mul_int(R, u64(mc), ovf);
                    const Rat rl = rat_sub(l, pl, ovf);
                    const unsigned short gn = (unsigned short)(S.gen[c] + 1);
                    if (DETAIL && lane == 0) {
                        ds_entity_rec& e = det.ent[n_ent];
                        e.origin = (unsigned short)c;
                        e.generation = gn;
                        e.part = 1;
                        e.launched = 1;
                        e.group = (unsigned short)gidx;
                        e.parallelism = mc;
                        e.load_num = (long long)pl.n;
                        e.load_den = (long long)pl.d;
                        e.exec_num = (long long)R.n;
                        e.exec_den = (long long)R.d;
                        e.res_num = (long long)rl.n;
                        e.res_den = (long long)rl.d;
                    }
                    __syncwarp();
                    if (lane == 0) {
                        S.gen[c] = gn;
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
                    ds_entity_rec& e = det.ent[n_ent + pos];
                    e.origin = (unsigned short)v;
                    e.generation = S.gen[v];
                    e.part = S.ppart[v];
                    e.launched = 0;
                    e.group = (unsigned short)gidx;
                    e.parallelism = S.mq[v];
                    e.load_num = (long long)S.pn[v];
                    e.load_den = (long long)S.pd[v];
                    e.exec_num = (long long)S.xn[v];
                    e.exec_den = (long long)S.xd[v];
                    e.res_num = 0;
                    e.res_den = 0;
                }
                ++pos;
            });
            if (lane == 0) {
                ds_group_rec& gr = det.grp[gidx];
                gr.resp_num = (long long)R.n;
                gr.resp_den = (long long)R.d;
                gr.spare_sms = spare0;
                gr.div_group = (unsigned short)g;
                gr.bottleneck = (unsigned short)(first_ent + n_launch + bott_pos);
                gr.first_entity = (unsigned short)first_ent;
                gr.n_launches = (unsigned short)n_launch;
                gr.n_members = (unsigned short)n_mem;
                gr.reserved = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) gr.unlaunched[k] = k < W ? (cands.w[k] & ~whole.w[k]) : 0;
            }
        }
        for (int v = lane; v < n; v += 32) {
            if (org.test(v)) S.done[v] = short(gidx);
        }
#pragma unroll
        for (int k = 0; k < W; ++k) done_mask.w[k] |= org.w[k] | whole.w[k];
        n_ent += n_mem;
        proposed = rat_add(proposed, R, ovf);
        ++gidx;
        __syncwarp();
    }
    {
        bool all = true;
#pragma unroll
        for (int k = 0; k < W; ++k) all &= done_mask.w[k] == V.w[k];
        if (!all) return DS_EINVARIANT;  // "scheduling finished with unplaced kernels"
    }
    bound[DS_BOUND_PROPOSED] = proposed;
    n_groups_out = gidx;
    n_ent_out = n_ent;
    return __any_sync(FULL, ovf) ? DS_EOVERFLOW : DS_OK;
}

struct K1Args {
    u64 n_dags;
    const u32* node_off;
    const u32* edge_off;
    const u64* load_num;
    const u64* load_den;
    const u32* edges;
    Plat plat;
    u32 mask;
    int32_t* status;
    int64_t* bounds;
    uint16_t* n_groups;
    // detail mode
    ds_scheme_out det;
};

template <int W, bool DETAIL>
__global__ void __launch_bounds__(128) k1_analyse(const K1Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpState<W>& S = reinterpret_cast<WarpState<W>*>(smem_raw)[wib];
    const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
    const u32 nbase = a.node_off[0], ebase = a.edge_off[0];  // offsets are relative to element 0
    for (u64 d = u64(blockIdx.x) * (blockDim.x >> 5) + wib; d < a.n_dags; d += warps) {
        const u32 n0 = a.node_off[d] - nbase, n1 = a.node_off[d + 1] - nbase;
        const u32 e0 = a.edge_off[d] - ebase, e1 = a.edge_off[d + 1] - ebase;
        const int n = int(n1 - n0);
        // size classes: the W-word kernel takes 64*(W/4)... < n <= 64*W (W=1: n <= 64)
        if (W > 1 && n <= 64) continue;
        if (W == 1 && n > 64 && n <= DS_MAX_NODES) continue;
        Rat bound[DS_N_BOUNDS];
#pragma unroll
        for (int k = 0; k < DS_N_BOUNDS; ++k) bound[k] = Rat{0, 0};
        int ng = 0, nent = 0, ndiv = 0;
        DetailOut det{};
        if (DETAIL) {
            det.ent = a.det.entities + 2ull * n0;
            det.grp = a.det.groups + n0;
            det.node_block = a.det.node_block + n0;
            det.node_div_group = a.det.node_div_group + n0;
        }
        int st = analyse_dag<W, DETAIL>(S, lane, n, a.load_num + n0, a.load_den ? a.load_den + n0 : nullptr,
                                        a.edges + e0, int(e1 - e0), a.plat, a.mask, bound, ng, det, nent,
                                        ndiv);
        // canonical results must fit the ABI's int64 slots
        if (st == DS_OK) {
#pragma unroll
            for (int k = 0; k < DS_N_BOUNDS; ++k) {
                if (((bound[k].n | bound[k].d) >> 63) != 0) st = DS_EOVERFLOW;
            }
        }
        int64_t* b = (DETAIL ? a.det.bounds : a.bounds) + 10 * d;
        if (lane < 10) {
            const int k = lane >> 1;
            const u64 v = st == DS_OK ? ((lane & 1) ? bound[k].d : bound[k].n) : 0;
            b[lane] = (long long)v;
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
}

}  // namespace ds

// K6 — batched simulate_greedy (simulator.cpp:96-190): the work-conserving
// hardware-style dispatch the paper compares against (every kernel asks for
// min(m^max, M) SMs and starts as soon as its predecessors are done and enough
// SMs are free; simultaneously ready kernels start in release order, ties by a
// seeded shuffle (random) or by id (fifo)).
//
// One thread per (DAG, run); run r uses policy seed policy_seed + r (the
// run_benchmarks convention, experiment.cpp:271-276). Exact rational times in
// word type T: u64 first, a run that overflows is redone in u128 (k6_greedy
// with T = u128 over the runs flagged kK6Retry). The event loop is the
// reference's:
//   init, per node in id order: m = min(max_parallelism(load), M),
//        duration = exec_time(load, m) * factor (FactorSource, scaled mode:
//        uniform_int_distribution<long long>(lo, hi) / 1024 over mt19937_64)
//   release(source, 0); dispatch();
//   while running: t = min finish; pop every (finish == t) in id order,
//        free their SMs; for each popped v (id order), each successor s
//        ascending: if --preds_left[s] == 0 release(s, t) (random policy: the
//        tie rank is the next raw mt19937_64 output); dispatch()
//   dispatch: ready sorted by (release, tie, id); start each that fits.
// The factor stream is drawn completely before the first policy draw, so one
// generator state serves both (re-seeded in between).
#pragma once

#include "../../include/dagsched_b200.h"
#include "rat.cuh"
#include "rng.cuh"

#include <type_traits>

namespace ds {

constexpr int32_t kK6Retry = -2000;

struct K6Args {
    u64 n_dags;
    int runs;
    const u32* node_off;  // rebased
    const u32* edge_off;
    const u64* load_num;
    const u64* load_den;  // may be null
    const u32* edges;
    int M;
    u64 tmin_n, tmin_d;
    int policy;  // 0 fifo, 1 random
    u64 policy_seed;
    int scaled;
    u64 time_seed;
    long long lo, hi;  // factor grid bounds (FactorSource), scaled mode
    int32_t* status;   // [n_dags * runs]
    int64_t* makespan; // [n_dags * runs * 2]
    int64_t* events;   // optional [N * runs * 4]: start n/d, finish n/d
    unsigned char* scratch;  // n > 256: per-thread run state (K6Big), kK6BigThreads slots
};

// Per-run state: local arrays (n <= 256) or one HBM slot per thread (n <= 1024)
template <int NMAX, class T>
struct K6Local {
    static constexpr int NW = NMAX / 64;
    u64 succ[NMAX][NW];
    RatT<T> dur[NMAX], rel[NMAX], fin[NMAX];
    int m[NMAX];
    u64 tie[NMAX];
    unsigned short left[NMAX];
    static constexpr size_t kBytes = 0;
    __device__ __forceinline__ void bind(unsigned char*) {}
};
template <int NMAX, class T>
struct K6Slot {
    static constexpr int NW = NMAX / 64;
    u64 (*succ)[NW];
    RatT<T>*dur, *rel, *fin;
    int* m;
    u64* tie;
    unsigned short* left;
    static constexpr size_t kBytes = size_t(NMAX) * (NW * 8 + 3 * sizeof(RatT<T>) + 4 + 8 + 2);
    __device__ __forceinline__ void bind(unsigned char* base) {
        succ = reinterpret_cast<u64(*)[NW]>(base);
        base += size_t(NMAX) * NW * 8;
        dur = reinterpret_cast<RatT<T>*>(base);
        rel = dur + NMAX;
        fin = rel + NMAX;
        base += size_t(NMAX) * 3 * sizeof(RatT<T>);
        tie = reinterpret_cast<u64*>(base);
        m = reinterpret_cast<int*>(tie + NMAX);
        left = reinterpret_cast<unsigned short*>(m + NMAX);
    }
};
constexpr int kK6BigThreads = 148 * 32;  // resident threads of the n > 256 kernels (one HBM slot each)

template <class T>
__device__ __forceinline__ bool fits_i64_any(T v) {
    return (v >> 63) == 0;
}

template <class T>
__device__ __forceinline__ bool q_less(const RatT<T>& a, const RatT<T>& b) {
    return rat_cmp(a, b) < 0;
}

// Size classes: NMAX = 64 takes n <= 64, 256 takes 64 < n <= 256, 1024 (HBM
// slots) takes the rest (n > 1024: DS_ETOOBIG); the u128 passes take the runs
// of their class flagged kK6Retry.
template <int NMAX, class T>
__global__ void __launch_bounds__(64) k6_greedy(const K6Args a) {
    constexpr int NW = NMAX / 64;
    constexpr bool kSlot = NMAX > 256;
    const u64 total = a.n_dags * u64(a.runs);
    const u64 tid = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    using Arr = typename std::conditional<kSlot, K6Slot<NMAX, T>, K6Local<NMAX, T>>::type;
    for (u64 p = tid; p < total; p += u64(gridDim.x) * blockDim.x) {
        const u64 d = p / u64(a.runs);
        const int run = int(p - d * u64(a.runs));
        const u32 n0 = a.node_off[d] - a.node_off[0];
        const int n = int(a.node_off[d + 1] - a.node_off[d]);
        const bool mine = sizeof(T) == 16 ? (NMAX == 256 ? n <= 256 : n > 256)
                                          : (NMAX == 64 ? n <= 64 : NMAX == 256 ? (n > 64 && n <= 256) : n > 256);
        if (!mine) continue;  // another class
        if (sizeof(T) == 16 && a.status[p] != kK6Retry) continue;
        int st = DS_OK;
        if (n <= 0) st = DS_E_EMPTY;
        if (n > NMAX) st = DS_ETOOBIG;
        bool ovf = false;
        Arr A;
        A.bind(a.scratch + tid * Arr::kBytes);
        auto& succ = A.succ;
        auto& dur = A.dur;
        auto& rel = A.rel;
        auto& fin = A.fin;
        auto& m = A.m;
        auto& tie = A.tie;
        auto& left = A.left;
        const PlatT<T> P{a.M, RatT<T>{T(a.tmin_n), T(a.tmin_d)}};
        Mt64 g;
        if (st == DS_OK) {
            for (int v = 0; v < n; ++v) {
                for (int w = 0; w < NW; ++w) succ[v][w] = 0;
                left[v] = 0;
            }
            const u32 e0 = a.edge_off[d] - a.edge_off[0], e1 = a.edge_off[d + 1] - a.edge_off[0];
            for (u32 e = e0; e < e1; ++e) {
                const int u = int(a.edges[e] >> 16), v = int(a.edges[e] & 0xffff);
                if (u >= n || v >= n || u == v) {
                    st = DS_E_EDGE;
                    break;
                }
                const u64 bit = 1ull << (v & 63);
                if (!(succ[u][v >> 6] & bit)) {  // duplicates collapse as in DagTask::make
                    succ[u][v >> 6] |= bit;
                    ++left[v];
                }
            }
        }
        if (st == DS_OK && a.scaled) g.seed(a.time_seed);
        int src = -1, n_src = 0;
        for (int v = 0; st == DS_OK && v < n; ++v) {
            long long ln = (long long)a.load_num[n0 + v], ldn = a.load_den ? (long long)a.load_den[n0 + v] : 1;
            if (ldn < 0) {
                ln = -ln;
                ldn = -ldn;
            }
            if (ln <= 0 || ldn <= 0) {
                st = DS_E_LOAD;
                break;
            }
            const RatT<T> l = rat_reduce(T(u64(ln)), T(u64(ldn)));
            const int mp = max_par(l, P, ovf);
            m[v] = mp < a.M ? mp : a.M;
            RatT<T> t = exec_time(l, m[v], P, ovf);
            if (a.scaled) {  // factors.next() per node in id order (simulator.cpp:113-118)
                const long long k = uniform_ll(g, a.lo, a.hi);
                t = rat_mul(t, rat_reduce(T(u64(k)), T(1024)), ovf);
            }
            dur[v] = t;
            if (left[v] == 0) {
                src = v;
                ++n_src;
            }
        }
        if (st == DS_OK && n_src != 1) st = DS_E_SOURCES;
        if (st != DS_OK) {
            a.status[p] = st;
            a.makespan[2 * p] = 0;
            a.makespan[2 * p + 1] = 0;
            continue;
        }
        if (a.policy) g.seed(a.policy_seed + u64(run));
        u64 ready[NW], running[NW];
        for (int w = 0; w < NW; ++w) ready[w] = running[w] = 0;
        int free_sms = a.M, n_done = 0;
        RatT<T> now{0, 1};
        auto release = [&](int v, RatT<T> t) {
            rel[v] = t;
            tie[v] = a.policy ? g.next() : 0ull;
            ready[v >> 6] |= 1ull << (v & 63);
        };
        auto dispatch = [&]() {
            // visit ready nodes in (release, tie, id) order; start each that fits
            u64 seen[NW];
            for (int w = 0; w < NW; ++w) seen[w] = 0;
            for (;;) {
                int best = -1;
                for (int w = 0; w < NW; ++w) {
                    for (u64 x = ready[w] & ~seen[w]; x; x &= x - 1) {
                        const int v = w * 64 + __ffsll(x) - 1;
                        if (best < 0) {
                            best = v;
                            continue;
                        }
                        const int c = rat_cmp(rel[v], rel[best]);
                        if (c < 0 || (c == 0 && tie[v] < tie[best])) best = v;  // ascending v: id ties keep best
                    }
                }
                if (best < 0) break;
                seen[best >> 6] |= 1ull << (best & 63);
                if (m[best] <= free_sms) {
                    free_sms -= m[best];
                    ready[best >> 6] &= ~(1ull << (best & 63));
                    running[best >> 6] |= 1ull << (best & 63);
                    fin[best] = rat_add(now, dur[best], ovf);
                    if (a.events) {
                        int64_t* ev = a.events + (u64(n0 + best) * u64(a.runs) + u64(run)) * 4;
                        ev[0] = (long long)now.n;
                        ev[1] = (long long)now.d;
                        ev[2] = (long long)fin[best].n;
                        ev[3] = (long long)fin[best].d;
                    }
                }
            }
        };
        release(src, now);
        dispatch();
        for (;;) {
            int first = -1;
            for (int w = 0; w < NW; ++w) {
                for (u64 x = running[w]; x; x &= x - 1) {
                    const int v = w * 64 + __ffsll(x) - 1;
                    if (first < 0 || q_less(fin[v], fin[first])) first = v;
                }
            }
            if (first < 0 || ovf) break;
            const RatT<T> t = fin[first];
            now = t;
            u64 popped[NW];
            for (int w = 0; w < NW; ++w) {
                popped[w] = 0;
                for (u64 x = running[w]; x; x &= x - 1) {
                    const int v = w * 64 + __ffsll(x) - 1;
                    if (rat_cmp(fin[v], t) == 0) popped[w] |= 1ull << (v & 63);
                }
                running[w] &= ~popped[w];
            }
            for (int w = 0; w < NW; ++w) {
                for (u64 x = popped[w]; x; x &= x - 1) {
                    const int v = w * 64 + __ffsll(x) - 1;
                    free_sms += m[v];
                    ++n_done;
                }
            }
            for (int w = 0; w < NW; ++w) {
                for (u64 x = popped[w]; x; x &= x - 1) {
                    const int v = w * 64 + __ffsll(x) - 1;
                    for (int w2 = 0; w2 < NW; ++w2) {
                        for (u64 y = succ[v][w2]; y; y &= y - 1) {
                            const int s = w2 * 64 + __ffsll(y) - 1;
                            if (--left[s] == 0) release(s, t);
                        }
                    }
                }
            }
            dispatch();
        }
        if (ovf) {
            a.status[p] = sizeof(T) == 16 ? DS_EOVERFLOW : kK6Retry;
            a.makespan[2 * p] = 0;
            a.makespan[2 * p + 1] = 0;
            continue;
        }
        bool any_ready = false;
        for (int w = 0; w < NW; ++w) any_ready |= ready[w] != 0;
        if (any_ready) st = DS_EINVARIANT;        // "greedy simulation stalled with ready kernels"
        else if (n_done != n) st = DS_E_CYCLE;    // unreachable nodes: not a DAG DagTask::make accepts
        const bool fits = fits_i64_any(now.n) && fits_i64_any(now.d);
        if (st == DS_OK && !fits) st = DS_EOVERFLOW;
        a.status[p] = st;
        a.makespan[2 * p] = st == DS_OK ? (long long)now.n : 0;
        a.makespan[2 * p + 1] = st == DS_OK ? (long long)now.d : 0;
    }
}

}  // namespace ds

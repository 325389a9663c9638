// K2 — node workload kernels (sm_100a), the GPU kernels a schedule executes.
//
// The paper emulates node loads with one kernel "with various iteration
// counts"; the reference ships no GPU code. Here every node is
// a memory-bound streaming kernel whose element count is proportional to its
// load, so its duration on m SMs follows Eq. 1 (C = load/m, floored at t_min)
// once the time unit is calibrated (bench_executor.py).
//
// Each CTA processes one contiguous slice of the entity's element range and
// stamps %globaltimer at entry and exit plus %smid. One CTA per SM is forced by
// the dynamic shared-memory footprint (> half of an SM's 228 KB), so an entity
// launched with grid = m holds exactly m SMs — the quota the scheduler gave it.
//
// Variants:
//   k2_mix        LDG.128/STG.128, 4 independent 16-B loads in flight per
//                 thread per iteration (8 B/elem algorithmic traffic)
//   k2_axpy       fp32 y = a*x + y, no FMA contraction (12 B/elem)
//   k2_mix_tma    warp-specialised cp.async.bulk (TMA engine) ring, below
#pragma once

#include <cstdint>

namespace ds {

struct NodeArgs {
    const uint32_t* x;
    uint32_t* y;
    unsigned long long lo, hi;  // element range of this entity
    unsigned long long* stamps; // [replay][total][2]
    uint32_t* smids;            // [replay][total]
    unsigned long long* span;   // [replay][2]: min start, max end
    const int* replay;          // replay index (< 0: warm-up, not recorded)
    uint32_t slot;              // first CTA slot of this entity
    uint32_t total;             // CTAs per replay
    float a;                    // axpy coefficient
    int cap;                    // recorded replays (bound on *replay)
};

constexpr int kNodeSmem = 120 * 1024;  // > 114 KB: at most one node CTA per SM

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}

// lowbias32 (an integer avalanche hash); host twin in executor.py
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t v) {
    v ^= v >> 16;
    v *= 0x7feb352du;
    v ^= v >> 15;
    v *= 0x846ca68bu;
    v ^= v >> 16;
    return v;
}

__device__ __forceinline__ void cta_slice(const NodeArgs& a, unsigned long long& s0, unsigned long long& s1) {
    const unsigned long long len = a.hi - a.lo;
    s0 = a.lo + len * blockIdx.x / gridDim.x;
    s1 = a.lo + len * (blockIdx.x + 1) / gridDim.x;
}

__device__ __forceinline__ void stamp_exit(const NodeArgs& a, unsigned long long t0) {
    if (threadIdx.x != 0) return;
    const unsigned long long t1 = gtimer();
    const int r = *a.replay;
    if (r < 0 || r >= a.cap) return;
    const unsigned long long idx = (unsigned long long)r * a.total + a.slot + blockIdx.x;
    if (a.stamps) {
        a.stamps[2 * idx] = t0;
        a.stamps[2 * idx + 1] = t1;
    }
    if (a.smids) a.smids[idx] = smid();
    atomicMin(&a.span[2 * r], t0);
    atomicMax(&a.span[2 * r + 1], t1);
}

// y[s0, s1) = mix(x[s0, s1)) with LDG.128/STG.128, U independent 16-B loads
// in flight per thread per iteration (1024 threads: U x 16 KB per SM).
template <int U>
__device__ __forceinline__ void mix_ldg_slice(const uint32_t* x, uint32_t* y, unsigned long long s0,
                                              unsigned long long s1) {
    // scalar head/tail, 16-byte vectors in between (buffers are 256-B aligned)
    const unsigned long long v0 = (s0 + 3) >> 2, v1 = s1 >> 2;
    if (v0 >= v1) {
        for (unsigned long long i = s0 + threadIdx.x; i < s1; i += blockDim.x) y[i] = mix32(__ldg(x + i));
        return;
    }
    for (unsigned long long i = s0 + threadIdx.x; i < (v0 << 2); i += blockDim.x) y[i] = mix32(__ldg(x + i));
    for (unsigned long long i = (v1 << 2) + threadIdx.x; i < s1; i += blockDim.x) y[i] = mix32(__ldg(x + i));
    const uint4* x4 = reinterpret_cast<const uint4*>(x);
    uint4* y4 = reinterpret_cast<uint4*>(y);
    const unsigned long long step = blockDim.x;
    unsigned long long i = v0 + threadIdx.x;
#define DS_MIX4(r) r.x = mix32(r.x), r.y = mix32(r.y), r.z = mix32(r.z), r.w = mix32(r.w)
    for (; i + (U - 1) * step < v1; i += U * step) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = __ldcs(x4 + i + u * step);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            DS_MIX4(r[u]);
            __stcs(y4 + i + u * step, r[u]);
        }
    }
    for (; i < v1; i += step) {
        uint4 r = __ldcs(x4 + i);
        DS_MIX4(r);
        __stcs(y4 + i, r);
    }
#undef DS_MIX4
}

template <int U>
__global__ void __launch_bounds__(1024, 1) k2_mix(const NodeArgs a) {
    __shared__ unsigned long long t0s;
    if (threadIdx.x == 0) t0s = gtimer();
    unsigned long long s0, s1;
    cta_slice(a, s0, s1);
    mix_ldg_slice<U>(a.x, a.y, s0, s1);
    __syncthreads();
    stamp_exit(a, t0s);
}

__global__ void __launch_bounds__(1024, 1) k2_axpy(const NodeArgs a) {
    __shared__ unsigned long long t0s;
    if (threadIdx.x == 0) t0s = gtimer();
    unsigned long long s0, s1;
    cta_slice(a, s0, s1);
    const float* x = reinterpret_cast<const float*>(a.x);
    float* y = reinterpret_cast<float*>(a.y);
    const float k = a.a;
    const unsigned long long v0 = (s0 + 3) >> 2, v1 = s1 >> 2;
    auto one = [&](unsigned long long i) { y[i] = __fadd_rn(__fmul_rn(k, x[i]), y[i]); };
    if (v0 >= v1) {
        for (unsigned long long i = s0 + threadIdx.x; i < s1; i += blockDim.x) one(i);
    } else {
        for (unsigned long long i = s0 + threadIdx.x; i < (v0 << 2); i += blockDim.x) one(i);
        for (unsigned long long i = (v1 << 2) + threadIdx.x; i < s1; i += blockDim.x) one(i);
        const float4* x4 = reinterpret_cast<const float4*>(x);
        float4* y4 = reinterpret_cast<float4*>(y);
        const unsigned long long step = blockDim.x;
        unsigned long long i = v0 + threadIdx.x;
        for (; i + step < v1; i += 2 * step) {
            const float4 p0 = __ldcs(x4 + i), p1 = __ldcs(x4 + i + step);
            float4 q0 = __ldcs(y4 + i), q1 = __ldcs(y4 + i + step);
#define DS_AXPY4(p, q)                     \
    q.x = __fadd_rn(__fmul_rn(k, p.x), q.x); \
    q.y = __fadd_rn(__fmul_rn(k, p.y), q.y); \
    q.z = __fadd_rn(__fmul_rn(k, p.z), q.z); \
    q.w = __fadd_rn(__fmul_rn(k, p.w), q.w)
            DS_AXPY4(p0, q0);
            DS_AXPY4(p1, q1);
            __stcs(y4 + i, q0);
            __stcs(y4 + i + step, q1);
        }
        for (; i < v1; i += step) {
            const float4 p = __ldcs(x4 + i);
            float4 q = __ldcs(y4 + i);
            DS_AXPY4(p, q);
            __stcs(y4 + i, q);
        }
#undef DS_AXPY4
    }
    __syncthreads();
    stamp_exit(a, t0s);
}

// ------------------------------------------------ TMA bulk-copy staged variant
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------ warp-specialised TMA streaming variant
// One producer warp (one elected lane) streams the CTA's slice through a
// ring of kTmaStages x kTmaChunk shared-memory stages with cp.async.bulk
// (TMA engine, completion on the stage's `full` mbarrier); kTmaConsumerWarps
// consumer warps transform each stage (LDS.128 -> mix -> STG.128 streaming
// stores) and release it on its `empty` mbarrier (one arrival per warp). No
// CTA-wide barrier in the steady state, and up to kTmaStages x 32 KB of reads
// in flight per SM without holding registers — what a lone node (a few SMs
// busy, the critical path of a DAG) needs to go beyond the ~64 KB an LDG loop
// keeps in flight. The 192 KB ring also forces one CTA per SM.
constexpr int kTmaStages = 6;
constexpr int kTmaChunk = 32 * 1024;
constexpr int kTmaConsumerWarps = 16;
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;
constexpr int kTmaSmem = kTmaStages * kTmaChunk;

struct TmaRing {
    uint64_t full[kTmaStages];
    uint64_t empty[kTmaStages];
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_ring_init(TmaRing* r) {  // one thread, then a CTA barrier
    for (int s = 0; s < kTmaStages; ++s) {
        mbar_init(&r->full[s], 1);
        mbar_init(&r->empty[s], kTmaConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// y[s0, s1) = mix(x[s0, s1)) by the whole CTA (kTmaThreads threads). `it`
// counts the ring's chunks used so far by this CTA (identical in every
// thread), so a persistent CTA can call this once per work item.
__device__ __forceinline__ void tma_mix_slice(const uint32_t* x, uint32_t* y, unsigned long long s0,
                                              unsigned long long s1, unsigned char* sm, TmaRing* ring,
                                              uint32_t& it) {
    const unsigned long long v0 = (s0 + 3) >> 2, v1 = s1 >> 2;  // 16-B aligned interior
    if (v0 >= v1) {
        for (unsigned long long i = s0 + threadIdx.x; i < s1; i += blockDim.x) y[i] = mix32(__ldg(x + i));
        return;
    }
    for (unsigned long long i = s0 + threadIdx.x; i < (v0 << 2); i += blockDim.x) y[i] = mix32(__ldg(x + i));
    for (unsigned long long i = (v1 << 2) + threadIdx.x; i < s1; i += blockDim.x) y[i] = mix32(__ldg(x + i));
    constexpr unsigned long long kChunkV = kTmaChunk / 16;  // uint4 per stage
    const unsigned long long nv = v1 - v0;
    const uint32_t n_chunks = uint32_t((nv + kChunkV - 1) / kChunkV);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint4* x4 = reinterpret_cast<const uint4*>(x) + v0;
    uint4* y4 = reinterpret_cast<uint4*>(y) + v0;
    if (warp == kTmaConsumerWarps) {  // producer
        if (lane == 0) {
            for (uint32_t c = 0; c < n_chunks; ++c) {
                const uint32_t idx = it + c, s = idx % kTmaStages, k = idx / kTmaStages;
                if (k > 0) mbar_wait(&ring->empty[s], (k - 1) & 1);
                const unsigned long long nc = min(kChunkV, nv - c * kChunkV);
                mbar_expect_tx(&ring->full[s], uint32_t(nc * 16));
                bulk_g2s(sm + s * kTmaChunk, x4 + c * kChunkV, uint32_t(nc * 16), &ring->full[s]);
            }
        }
    } else {
        const int t = threadIdx.x;  // < kTmaConsumerWarps * 32
        for (uint32_t c = 0; c < n_chunks; ++c) {
            const uint32_t idx = it + c, s = idx % kTmaStages, k = idx / kTmaStages;
            const unsigned long long nc = min(kChunkV, nv - c * kChunkV);
            mbar_wait(&ring->full[s], k & 1);
            const uint4* buf = reinterpret_cast<const uint4*>(sm + s * kTmaChunk);
            uint4* dst = y4 + c * kChunkV;
#pragma unroll 4
            for (unsigned long long i = t; i < nc; i += kTmaConsumerWarps * 32) {
                uint4 r = buf[i];
                r.x = mix32(r.x), r.y = mix32(r.y), r.z = mix32(r.z), r.w = mix32(r.w);
                __stcs(dst + i, r);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ring->empty[s]);
        }
    }
    it += n_chunks;
}

__global__ void __launch_bounds__(kTmaThreads, 1) k2_mix_tma(const NodeArgs a) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ TmaRing ring;
    __shared__ unsigned long long t0s;
    if (threadIdx.x == 0) {
        t0s = gtimer();
        tma_ring_init(&ring);
    }
    __syncthreads();
    unsigned long long s0, s1;
    cta_slice(a, s0, s1);
    uint32_t it = 0;
    tma_mix_slice(a.x, a.y, s0, s1, sm, &ring, it);
    __syncthreads();
    stamp_exit(a, t0s);
}

__global__ void k2_init(uint32_t* x, unsigned long long n, uint32_t seed, int fp, uint32_t* y) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint32_t h = mix32(uint32_t(i) ^ mix32(seed ^ uint32_t(i >> 32) * 0x9e3779b9u));
        if (fp) {
            // floats in [-1, 1): 24 random mantissa bits, exactly representable
            reinterpret_cast<float*>(x)[i] = float(int(h >> 8) - (1 << 23)) * (1.0f / float(1 << 23));
            reinterpret_cast<float*>(y)[i] = float(int(mix32(h) >> 8) - (1 << 23)) * (1.0f / float(1 << 23));
        } else {
            x[i] = h;
        }
    }
}

__global__ void k2_tick(int* replay) { *replay += 1; }

// acquire load of a completion counter (dependency hand-off)
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ------------------------------------------------ dynamic persistent engine
// One resident CTA per SM for the whole DAG, work-conserving, with look-ahead
// claiming. Per entity e (quota m_e, augmented-graph predecessors P(e)):
//   claimed[e]     ranks of e handed out so far (an entity is m_e items, so it
//                  never holds more than its quota of SMs; a CTA runs one item
//                  at a time, so concurrent entities sit on disjoint SMs);
//   pend_claim[e]  sum over P(e) of ranks not yet claimed;
//   pend_done[e]   sum over P(e) of ranks not yet finished.
// Warp 0 of an idle CTA scans the entities in plan order (= schedule
// priority), 32 per coalesced probe, and claims a rank of the first entity
// that can start (pend_done = 0) or, failing that, of the first whose
// predecessors are all claimed (pend_claim = 0) — then waits for its
// pend_done to reach 0. The claim round trip thus overlaps the predecessors'
// execution, and the dependency hand-off on the critical path is one fence +
// fire-and-forget reductions (RED) in the finishing CTA and one acquire poll
// in the waiting one, the same as a static CTA assignment, without its
// mis-placements. Deadlock-free: the earliest (topological) waiting rank has
// every predecessor rank claimed, hence running, hence finishing.
// With egroup (DS_PLAN_PRIORITY) the probe only considers entities of the
// group of the first entity that still has unclaimed ranks (`cur`; plans are
// in group order): group g+1 is not touched while a group-g rank is
// unclaimed, so every group-g entity finds its quota of CTAs, and CTAs that
// finish their group-g rank early move on to group g+1 instead of idling.
struct DEnt {
    const uint32_t* x;
    uint32_t* y;
    unsigned long long lo, hi;
    uint32_t m, slot, succ_off, n_succ, pred_ranks;
};
struct DArgs {
    const DEnt* ents;
    const uint32_t* succs;
    const uint32_t* quota;      // [n] m_e (read-only copy for the warp probes)
    const uint32_t* egroup;     // [n] group of e (DS_PLAN_PRIORITY), else nullptr
    uint32_t n, n_init;
    unsigned int* claimed;      // [n]
    unsigned int* pend_claim;   // [n]
    unsigned int* pend_done;    // [n]
    unsigned int* idle;         // [1] stream engine: CTAs with nothing in flight
    unsigned int* next_chunk;   // [n] chunked ranks: next chunk of the entity
    unsigned long long chunk;   // elements per chunk, 0 = fixed slices
    int rec;                    // recorded replay slot, < 0: not recorded
    unsigned long long* stamps;
    uint32_t* smids;
    unsigned long long* span;
    uint32_t total;
};

__device__ __forceinline__ unsigned int ld_relaxed(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k3_dyn_reset(const DArgs a) {
    for (uint32_t i = threadIdx.x; i < a.n; i += blockDim.x) {
        a.claimed[i] = 0;
        a.pend_claim[i] = a.ents[i].pred_ranks;
        a.pend_done[i] = a.ents[i].pred_ranks;
        if (a.next_chunk) a.next_chunk[i] = 0;
    }
    if (threadIdx.x == 0 && a.idle) *a.idle = 0;
}

// One probe pass of a warp over the plan from `cur`: claims a rank of the
// first entity that can start (pend_done = 0), else of the first whose
// predecessors are all claimed (pend_claim = 0), window by window; ent = ~0u
// when nothing is open now. Advances `cur` past fully handed-out entities.
// (Measured: looking for a startable rank in every window before reserving
// one is no faster, at M = 148, 32 or 8.)
__device__ __forceinline__ void dyn_probe(const DArgs& a, const int lane, uint32_t& cur, uint32_t& ent,
                                          uint32_t& rank) {
    ent = ~0u;
    rank = 0;
    bool got = false;
    uint32_t gcur = ~0u;  // group of `cur` (priority plans)
    bool stop = false;
#pragma unroll 1
    for (uint32_t base = cur; base < a.n && !got && !stop; base += 32) {
        const uint32_t e = base + lane;
        const bool valid = e < a.n;
        const uint32_t m = valid ? __ldg(a.quota + e) : 0;
        const uint32_t cl = valid ? ld_relaxed(a.claimed + e) : 0;
        const uint32_t pc = valid ? ld_relaxed(a.pend_claim + e) : 1;
        const uint32_t pd = valid ? ld_relaxed(a.pend_done + e) : 1;
        bool open = valid && cl < m;
        const unsigned open_mask = __ballot_sync(~0u, open);
        if (base == cur) {
            cur = open_mask ? base + __ffs(open_mask) - 1 : base + 32;
            if (a.egroup && cur < a.n) gcur = __ldg(a.egroup + cur);
        }
        if (a.egroup) {  // later groups wait until this one is fully claimed
            const bool later = valid && __ldg(a.egroup + e) > gcur;
            open = open && !later;
            stop = __any_sync(~0u, later);  // plan order = group order: nothing after
        }
        unsigned pick = __ballot_sync(~0u, open && pc == 0 && pd == 0);
        if (!pick) pick = __ballot_sync(~0u, open && pc == 0);
        while (pick && !got) {
            const int l = __ffs(pick) - 1;
            pick &= pick - 1;
            uint32_t c = 0;
            if (lane == l) c = atomicAdd(a.claimed + e, 1u);
            c = __shfl_sync(~0u, c, l);
            const uint32_t ml = __shfl_sync(~0u, m, l);
            if (c < ml) {
                got = true;
                ent = base + l;
                rank = c;
            }
        }
    }
}

// a claimed rank of `ent` counts as claimed for its successors (lane 0)
__device__ __forceinline__ void dyn_commit(const DArgs& a, uint32_t ent) {
    const DEnt& d = a.ents[ent];
    for (uint32_t k = 0; k < d.n_succ; ++k) atomicSub(a.pend_claim + a.succs[d.succ_off + k], 1u);
}

// kAhead (TMA ring, fixed slices): the producer warp schedules — once it has
// issued an item's last load it already claims the CTA's next item while the
// consumer warps drain the ring, so the claim's round trips leave the gap
// between items (the rank still waits for its predecessors after the item
// ends; deadlock-free as before: the earliest claimed-but-waiting rank has
// every predecessor rank claimed, and claimed ranks ahead of it are running).
template <bool kTma, bool kAhead = false>
__global__ void __launch_bounds__(kTma ? kTmaThreads : 1024, 1) k3_dynamic(const DArgs a) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ TmaRing ring;
    __shared__ unsigned long long t0s;
    __shared__ uint32_t s_ent, s_rank, s_chunk;
    if (kTma && threadIdx.x == 0) tma_ring_init(&ring);
    constexpr int kSched = (kTma && kAhead) ? kTmaConsumerWarps : 0;  // the scheduling warp
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t it = 0;   // TMA ring chunks used by this CTA
    uint32_t cur = 0;  // entities before cur are fully handed out (scheduling warp)
    uint32_t next_ent = ~0u, next_rank = 0;  // claimed ahead (kAhead)
#pragma unroll 1
    while (true) {
        if (warp == kSched) {
            uint32_t ent = next_ent, rank = next_rank;
            next_ent = ~0u;
            while (ent == ~0u && cur < a.n) {
                dyn_probe(a, lane, cur, ent, rank);
                if (ent != ~0u) {
                    if (lane == 0) dyn_commit(a, ent);
                    break;
                }
                __nanosleep(32);
            }
            if (lane == 0 && ent != ~0u) {
                while (ld_acquire(a.pend_done + ent) != 0) {
                }  // tight: every reserved rank of ent starts within one L2 round trip
                t0s = gtimer();
            }
            if (lane == 0) {
                s_ent = ent;
                s_rank = rank;
            }
        }
        __syncthreads();
        const uint32_t ent = s_ent, rank = s_rank;
        const unsigned long long my_t0 = t0s;
        if (ent == ~0u) break;
        const DEnt e = a.ents[ent];
        const unsigned long long len = e.hi - e.lo;
        if (a.chunk == 0) {
            const unsigned long long s0 = e.lo + len * rank / e.m, s1 = e.lo + len * (rank + 1) / e.m;
            if constexpr (kTma) tma_mix_slice(e.x, e.y, s0, s1, sm, &ring, it);
            else mix_ldg_slice<4>(e.x, e.y, s0, s1);
            if (kAhead && warp == kSched && cur < a.n) {  // loads issued: claim the next item now
                dyn_probe(a, lane, cur, next_ent, next_rank);
                if (next_ent != ~0u && lane == 0) dyn_commit(a, next_ent);
            }
        } else {
            // chunked ranks: claim chunk after chunk of the entity's range; the
            // next claim is issued before the current chunk is processed
            const unsigned long long nch = (len + a.chunk - 1) / a.chunk;
            if (threadIdx.x == 0) s_chunk = atomicAdd(a.next_chunk + ent, 1u);
            __syncthreads();
            unsigned long long c = s_chunk;
#pragma unroll 1
            while (c < nch) {
                __syncthreads();  // every thread has read s_chunk
                if (threadIdx.x == 0) s_chunk = atomicAdd(a.next_chunk + ent, 1u);
                const unsigned long long s0 = e.lo + c * a.chunk, s1 = min(e.hi, s0 + a.chunk);
                if constexpr (kTma) tma_mix_slice(e.x, e.y, s0, s1, sm, &ring, it);
                else mix_ldg_slice<4>(e.x, e.y, s0, s1);
                __syncthreads();
                c = s_chunk;
            }
        }
        __syncthreads();
        // completion in warp 1 while warp 0 already claims the next item: the
        // fence (waits for this CTA's stores, observed through the barrier)
        // overlaps the claim's round trips
        if (threadIdx.x == 32) {
            const unsigned long long t0s = my_t0;
            const unsigned long long t1 = gtimer();
            __threadfence();  // this item's stores before its completion
            for (uint32_t k = 0; k < e.n_succ; ++k) atomicSub(a.pend_done + a.succs[e.succ_off + k], 1u);
            if (a.rec >= 0) {
                const unsigned long long idx = (unsigned long long)a.rec * a.total + e.slot + rank;
                if (a.stamps) {
                    a.stamps[2 * idx] = t0s;
                    a.stamps[2 * idx + 1] = t1;
                }
                if (a.smids) a.smids[idx] = smid();
                atomicMin(&a.span[2 * a.rec], t0s);
                atomicMax(&a.span[2 * a.rec + 1], t1);
            }
        }
    }
}

}  // namespace ds

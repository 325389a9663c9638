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
//   k2_mix_bulk   cp.async.bulk global->shared (TMA engine, mbarrier
//                 complete_tx) and shared->global bulk stores, 4-stage ring
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
constexpr int kBulkStages = 4;
constexpr int kBulkChunk = 24 * 1024;  // bytes per stage (4 x 24 KB ring)

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

__global__ void __launch_bounds__(1024, 1) k2_mix(const NodeArgs a) {
    __shared__ unsigned long long t0s;
    if (threadIdx.x == 0) t0s = gtimer();
    unsigned long long s0, s1;
    cta_slice(a, s0, s1);
    // scalar head/tail, 16-byte vectors in between (buffers are 256-B aligned)
    const unsigned long long v0 = (s0 + 3) >> 2, v1 = s1 >> 2;
    if (v0 >= v1) {
        for (unsigned long long i = s0 + threadIdx.x; i < s1; i += blockDim.x) a.y[i] = mix32(__ldg(a.x + i));
    } else {
        for (unsigned long long i = s0 + threadIdx.x; i < (v0 << 2); i += blockDim.x) a.y[i] = mix32(__ldg(a.x + i));
        for (unsigned long long i = (v1 << 2) + threadIdx.x; i < s1; i += blockDim.x) a.y[i] = mix32(__ldg(a.x + i));
        const uint4* x4 = reinterpret_cast<const uint4*>(a.x);
        uint4* y4 = reinterpret_cast<uint4*>(a.y);
        const unsigned long long step = blockDim.x;
        unsigned long long i = v0 + threadIdx.x;
        for (; i + 3 * step < v1; i += 4 * step) {
            uint4 r0 = __ldcs(x4 + i), r1 = __ldcs(x4 + i + step), r2 = __ldcs(x4 + i + 2 * step),
                  r3 = __ldcs(x4 + i + 3 * step);
#define DS_MIX4(r) r.x = mix32(r.x), r.y = mix32(r.y), r.z = mix32(r.z), r.w = mix32(r.w)
            DS_MIX4(r0);
            DS_MIX4(r1);
            DS_MIX4(r2);
            DS_MIX4(r3);
            __stcs(y4 + i, r0);
            __stcs(y4 + i + step, r1);
            __stcs(y4 + i + 2 * step, r2);
            __stcs(y4 + i + 3 * step, r3);
        }
        for (; i < v1; i += step) {
            uint4 r = __ldcs(x4 + i);
            DS_MIX4(r);
            __stcs(y4 + i, r);
        }
#undef DS_MIX4
    }
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

__global__ void __launch_bounds__(1024, 1) k2_mix_bulk(const NodeArgs a) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ unsigned long long t0s;
    __shared__ __align__(8) uint64_t bars[kBulkStages];
    if (threadIdx.x == 0) {
        t0s = gtimer();
        for (int s = 0; s < kBulkStages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long s0, s1;
    cta_slice(a, s0, s1);
    const unsigned long long v0 = (s0 + 3) >> 2, v1 = s1 >> 2;  // 16-B aligned interior
    if (v0 >= v1) {
        for (unsigned long long i = s0 + threadIdx.x; i < s1; i += blockDim.x) a.y[i] = mix32(__ldg(a.x + i));
    } else {
        for (unsigned long long i = s0 + threadIdx.x; i < (v0 << 2); i += blockDim.x) a.y[i] = mix32(__ldg(a.x + i));
        for (unsigned long long i = (v1 << 2) + threadIdx.x; i < s1; i += blockDim.x) a.y[i] = mix32(__ldg(a.x + i));
        const unsigned long long base = v0 << 2, n_el = (v1 - v0) << 2;  // elements in the interior
        constexpr unsigned long long kChunkEl = kBulkChunk / 4;
        const unsigned long long n_chunks = (n_el + kChunkEl - 1) / kChunkEl;
        auto issue = [&](unsigned long long c) {  // thread 0: load chunk c into stage c % S
            const int s = int(c % kBulkStages);
            const unsigned long long e0 = base + c * kChunkEl;
            const unsigned long long ne = min(kChunkEl, base + n_el - e0);
            mbar_expect_tx(&bars[s], uint32_t(ne * 4));
            bulk_g2s(sm + s * kBulkChunk, a.x + e0, uint32_t(ne * 4), &bars[s]);
        };
        if (threadIdx.x == 0) {
            for (unsigned long long c = 0; c < n_chunks && c < kBulkStages; ++c) issue(c);
        }
        for (unsigned long long c = 0; c < n_chunks; ++c) {
            const int s = int(c % kBulkStages);
            const unsigned long long e0 = base + c * kChunkEl;
            const unsigned long long ne = min(kChunkEl, base + n_el - e0);
            mbar_wait(&bars[s], uint32_t((c / kBulkStages) & 1));
            uint4* buf = reinterpret_cast<uint4*>(sm + s * kBulkChunk);
            for (unsigned long long i = threadIdx.x; i < ne / 4; i += blockDim.x) {
                uint4 r = buf[i];
                r.x = mix32(r.x), r.y = mix32(r.y), r.z = mix32(r.z), r.w = mix32(r.w);
                buf[i] = r;
            }
            fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk copy
            __syncthreads();
            if (threadIdx.x == 0) {
                bulk_s2g(a.y + e0, buf, uint32_t(ne * 4));
                bulk_commit();
                if (c + kBulkStages < n_chunks) {
                    // stage s is reloaded: its store must have finished reading smem
                    bulk_wait_read<0>();
                    issue(c + kBulkStages);
                }
            }
        }
        if (threadIdx.x == 0) bulk_wait_all();
    }
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

// ------------------------------------------------ persistent engine (K3)
// One CTA per SM for the whole DAG. CTA b walks items[item_off[b] ..
// item_off[b+1]) — (entity, rank) pairs in group order — waits until every
// predecessor entity has all of its CTAs done for this epoch (counters only
// grow: entity p is complete in epoch k when done[p] >= m_p * (k+1)), runs its
// slice of the entity's element range with the k2_mix body, then publishes
// completion (fence + atomicAdd). Deadlock-free: predecessors always sit in
// strictly earlier groups, and every CTA walks its items in group order.
struct PEnt {
    const uint32_t* x;
    uint32_t* y;
    unsigned long long lo, hi;
    uint32_t m, slot, pred_off, n_preds;
};
struct PItem {
    uint32_t ent, rank;
};
struct PArgs {
    const PEnt* ents;
    const uint32_t* preds;
    const uint32_t* item_off;
    const PItem* items;
    unsigned int* done;
    unsigned int epoch;
    int rec;  // recorded replay slot, < 0: not recorded
    unsigned long long* stamps;
    uint32_t* smids;
    unsigned long long* span;
    uint32_t total;
};

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(1024, 1) k3_persistent(const PArgs a) {
    __shared__ unsigned long long t0s;
    const uint32_t b = blockIdx.x;
#pragma unroll 1
    for (uint32_t it = a.item_off[b]; it < a.item_off[b + 1]; ++it) {
        const PItem w = a.items[it];
        const PEnt e = a.ents[w.ent];
        if (threadIdx.x == 0) {
            for (uint32_t k = 0; k < e.n_preds; ++k) {
                const uint32_t p = a.preds[e.pred_off + k];
                const unsigned int need = a.ents[p].m * (a.epoch + 1);
                while (ld_acquire(a.done + p) < need) __nanosleep(32);
            }
            t0s = gtimer();
        }
        __syncthreads();
        const unsigned long long len = e.hi - e.lo;
        const unsigned long long s0 = e.lo + len * w.rank / e.m, s1 = e.lo + len * (w.rank + 1) / e.m;
        const unsigned long long v0 = (s0 + 3) >> 2, v1 = s1 >> 2;
        if (v0 >= v1) {
            for (unsigned long long i = s0 + threadIdx.x; i < s1; i += blockDim.x) e.y[i] = mix32(__ldg(e.x + i));
        } else {
            for (unsigned long long i = s0 + threadIdx.x; i < (v0 << 2); i += blockDim.x) e.y[i] = mix32(__ldg(e.x + i));
            for (unsigned long long i = (v1 << 2) + threadIdx.x; i < s1; i += blockDim.x) e.y[i] = mix32(__ldg(e.x + i));
            const uint4* x4 = reinterpret_cast<const uint4*>(e.x);
            uint4* y4 = reinterpret_cast<uint4*>(e.y);
            const unsigned long long step = blockDim.x;
            unsigned long long i = v0 + threadIdx.x;
            for (; i + 3 * step < v1; i += 4 * step) {
                uint4 r0 = __ldcs(x4 + i), r1 = __ldcs(x4 + i + step), r2 = __ldcs(x4 + i + 2 * step),
                      r3 = __ldcs(x4 + i + 3 * step);
#define DS_MIX4(r) r.x = mix32(r.x), r.y = mix32(r.y), r.z = mix32(r.z), r.w = mix32(r.w)
                DS_MIX4(r0);
                DS_MIX4(r1);
                DS_MIX4(r2);
                DS_MIX4(r3);
                __stcs(y4 + i, r0);
                __stcs(y4 + i + step, r1);
                __stcs(y4 + i + 2 * step, r2);
                __stcs(y4 + i + 3 * step, r3);
            }
            for (; i < v1; i += step) {
                uint4 r = __ldcs(x4 + i);
                DS_MIX4(r);
                __stcs(y4 + i, r);
            }
#undef DS_MIX4
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long t1 = gtimer();
            if (a.rec >= 0) {
                const unsigned long long idx = (unsigned long long)a.rec * a.total + e.slot + w.rank;
                if (a.stamps) {
                    a.stamps[2 * idx] = t0s;
                    a.stamps[2 * idx + 1] = t1;
                }
                if (a.smids) a.smids[idx] = smid();
                atomicMin(&a.span[2 * a.rec], t0s);
                atomicMax(&a.span[2 * a.rec + 1], t1);
            }
            __threadfence();
            atomicAdd(a.done + w.ent, 1u);
        }
    }
}

}  // namespace ds

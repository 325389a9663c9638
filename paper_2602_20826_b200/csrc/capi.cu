// C-ABI entry points of libdagsched_b200.so (include/dagsched_b200.h).
//
// ds_analyze_batch       evaluate_corpus (experiment.cpp:52-79) + lower_bound
// ds_analyze_batch_multi the same, contiguous shards over several GPUs
// ds_schedule_batch      schedule() + build_blocks/build_groups detail
// ds_session_*           device-resident replay used by bench.py
//
// Host-pointer calls stream the batch through the GPU in chunks on three
// streams so the PCIe copies of chunk i+1 overlap the analysis of chunk i.
#include "../../include/dagsched_b200.h"
#include "k1_launch.h"

#include <cstdlib>

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <string>
#include <thread>
#include <vector>

namespace ds {

// k4_validate.cu
void k4_launch(u64 n_dags, const u32* node_off, const int32_t* status, const uint16_t* n_groups,
               const ds_group_rec* groups, const ds_entity_rec* ents, const int64_t* bounds, int samples,
               long long lo, long long hi, u64 seed, unsigned char* over, double* ratio, int32_t* st,
               cudaStream_t stream);

// k1_small.cu: the latency path (one kernel, zero-copy mapped buffers)
cudaError_t k1_small_configure();
cudaError_t k1_small_launch(const K1Args& a, bool detail, cudaStream_t s);

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define DS_CUDA(call)                                                                                   \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) return fail(DS_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

int check_platform(const ds_platform* p, PlatT<u64>& out) {
    if (!p) return fail(DS_EINVAL, "platform is NULL");
    if (p->sm_count < 1) return fail(DS_EINVAL, "sm_count must be >= 1");  // exec_model.hpp:14-18
    long long n = p->tmin_num, d = p->tmin_den;
    if (d == 0) return fail(DS_EINVAL, "t_min denominator is zero");
    if (d < 0) {
        n = -n;
        d = -d;
    }
    if (n <= 0) return fail(DS_EINVAL, "t_min must be positive");
    u64 a = u64(n), b = u64(d);
    while (b) {
        const u64 t = a % b;
        a = b;
        b = t;
    }
    if (p->flags & ~(DS_PF_MIN_LOAD_ONE | DS_PF_PREMADE)) return fail(DS_EINVAL, "unknown platform flags");
    out.M = p->sm_count;
    out.tmin = RatT<u64>{u64(n) / a, u64(d) / a};
    out.minl = (p->flags & DS_PF_PREMADE) ? 2 : ((p->flags & DS_PF_MIN_LOAD_ONE) ? 1 : 0);
    return DS_OK;
}

int configure(int device, bool detail, K1Occupancy& occ) {
    static std::mutex mu;
    static K1Occupancy cache[128];
    static bool ready[128] = {};
    std::lock_guard<std::mutex> lock(mu);
    const int slot = (device & 63) * 2 + (detail ? 1 : 0);
    if (ready[slot]) {
        occ = cache[slot];
        return DS_OK;
    }
    DS_CUDA(k1_configure(device, detail, occ));
    DS_CUDA(k1_small_configure());
    cache[slot] = occ;
    ready[slot] = true;
    return DS_OK;
}

// the largest DAG of DAGs [lo, hi): picks the size-class kernels k1_launch runs
u32 batch_max_n(const uint32_t* node_off, u64 lo, u64 hi) {
    u32 m = 0;
    for (u64 d = lo; d < hi; ++d) m = std::max(m, node_off[d + 1] - node_off[d]);
    return m;
}

// detail mode: DAG d's unlaunched-candidate masks start at word base[d] of
// ds_scheme_out::unlaunched (n_k * ceil(n_k / 64) words per earlier DAG k);
// returns the total word count
u64 unl_layout(const uint32_t* node_off, u64 n, u64* base) {
    u64 w = 0;
    for (u64 d = 0; d < n; ++d) {
        const u64 k = node_off[d + 1] - node_off[d];
        if (base) base[d] = w;
        w += k * ((k + 63) / 64);
    }
    return w;
}

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        bytes = std::max<size_t>(bytes, 16);
        if (bytes <= cap) return DS_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        DS_CUDA(cudaMalloc(&p, bytes));
        cap = bytes;
        return DS_OK;
    }
    template <class X>
    X* as() const {
        return static_cast<X*>(p);
    }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// ------------------------------------------------------ chunked host path
struct Slot {
    cudaStream_t s = nullptr;
    DevBuf node_off, edge_off, ln, ldn, edges, status, bounds, ngroups, retry, retry_count, handoff;
    DevBuf ln16, edges16;         // compact wire form staging (ds_analyze_batch16)
    DevBuf adj_off, adj, edge_cnt;  // triangular wire form staging (ds_analyze_batch_tri)
    DevBuf big_q, big_scratch;      // DAGs above 256 nodes (k1_big)
};

// ds_dag_batch16 -> the analysis' wide form, on the device (HBM-bound, tiny)
__global__ void k_widen16(const uint16_t* __restrict__ ln16, const uint16_t* __restrict__ e16, u64 nn, u64 ne,
                          u64* __restrict__ ln, u32* __restrict__ edges) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < nn; i += stride) ln[i] = ln16[i];
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < ne; i += stride) {
        const u32 e = e16[i];
        edges[i] = ((e >> 8) << 16) | (e & 0xffu);
    }
}

// pinned host staging (grows, never shrinks)
struct PinBuf {
    void* p = nullptr;
    void* dev = nullptr;  // device alias when mapped
    size_t cap = 0;
    int ensure(size_t bytes, bool mapped = false) {
        bytes = std::max<size_t>(bytes, 4096);
        if (bytes <= cap) return DS_OK;
        if (p) cudaFreeHost(p);
        p = dev = nullptr;
        cap = 0;
        DS_CUDA(cudaHostAlloc(&p, bytes, mapped ? cudaHostAllocMapped : cudaHostAllocDefault));
        if (mapped) DS_CUDA(cudaHostGetDevicePointer(&dev, p, 0));
        cap = bytes;
        return DS_OK;
    }
    PinBuf() = default;
    PinBuf(const PinBuf&) = delete;
    PinBuf& operator=(const PinBuf&) = delete;
    ~PinBuf() {
        if (p) cudaFreeHost(p);
    }
};

// Schedule-detail pass (ds_schedule_batch / ds_validate_batch): inputs and
// outputs each live in one device arena carved per call, crossing PCIe as ONE
// pinned copy each way, so a single-DAG call (the kept C++ API's schedule()
// and analyze()) costs one H2D, the K1 launches and one D2H — no allocation.
struct DetailView {
    u32 *node_off, *edge_off, *edges;
    u64 *ln, *ldn;
    int32_t* status;
    uint16_t *ne, *ng, *nd;
    int16_t *nb, *ndg;
    ds_entity_rec* ent;
    ds_group_rec* grp;
    int64_t* bounds;
    size_t out_bytes;
    uint64_t* unl;
    u64 unl_words;
    size_t o_status, o_ne, o_ng, o_nd, o_nb, o_ndg, o_ent, o_grp, o_bounds, o_unl;  // offsets in the out arena
};
struct DetailCtx {
    DevBuf in, out, retry, retry_count, k4_over, k4_ratio, k4_st, big_q, big_scratch;
    PinBuf in_stage, out_stage;
    DetailView v{};
};

constexpr int kMaxSlots = 8;
struct DeviceCtx {
    std::mutex mu;
    bool init = false;
    Slot slot[kMaxSlots];
    DevBuf retry, retry_count, handoff, big_q, big_scratch;  // scratch for the device-pointer entry point
    // host-batch pipeline (analyze_host): copy-in, front kernels, back
    // kernels, copy-out streams and per-slot events between them
    cudaStream_t pipe[6] = {};  // copy-in, front, back 0, copy-out, back 1, back 2
    cudaEvent_t pev[kMaxSlots][4] = {};
    bool pev_live[kMaxSlots] = {};  // slot's copy-out event recorded (buffers in use)
    DetailCtx det;
    PinBuf small_in, small_out;  // latency path: mapped (zero-copy) inputs and outputs
    DevBuf small_dev;            // latency path: device copy of the packed inputs
};

DeviceCtx& device_ctx(int dev);

// The slots' streams, in decreasing priority: slot k (the k-th chunk of a
// host batch) outranks every later slot, so when chunks overlap, the block
// scheduler serves the earliest chunk first and later chunks fill its tails
// (each K1 pass ends in a ~0.25 ms tail of long lane walks) instead of
// slowing it down. DS_STREAM_PRIO=0: equal priorities.
int create_slot_streams(DeviceCtx& ctx) {
    static const bool prio = [] {
        const char* e = getenv("DS_STREAM_PRIO");
        return !(e && e[0] == '0');
    }();
    int least = 0, greatest = 0;
    DS_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    for (int k = 0; k < kMaxSlots; ++k) {
        const int p = prio ? std::min(least, greatest + k) : least;
        DS_CUDA(cudaStreamCreateWithPriority(&ctx.slot[k].s, cudaStreamNonBlocking, p));
    }
    // pipeline: the back kernels (lane walks) outrank the next chunk's front
    // kernels, so a chunk's walks finish first and the front work fills
    // their tail
    const int pp[6] = {least, std::min(least, greatest + 1), greatest, least, greatest, greatest};
    for (int k = 0; k < 6; ++k) DS_CUDA(cudaStreamCreateWithPriority(&ctx.pipe[k], cudaStreamNonBlocking, pp[k]));
    for (auto& row : ctx.pev)
        for (auto& e : row) DS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx.init = true;
    return DS_OK;
}

// ------------------------------------------------------- latency path
// Host batches of at most kSmallDags DAGs go through k1_small (k1_small.cu):
// inputs packed into pinned memory and copied once, one launch, results read
// back from mapped pinned memory. DS_SMALL=0 disables it.
constexpr u64 kSmallDags = 64;
bool small_enabled() {
    static const bool on = [] {
        const char* e = getenv("DS_SMALL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// A host batch in either wire form, read element-wise for packing.
struct HostView {
    u64 n;
    const uint32_t *node_off, *edge_off;
    const int64_t *ln, *ld;     // wide form
    const uint16_t *ln16, *e16;  // compact form
    const uint32_t* edges;
    int64_t load(u64 i) const { return ln ? ln[i] : int64_t(ln16[i]); }
    uint32_t edge(u64 i) const { return edges ? edges[i] : ((uint32_t(e16[i]) >> 8) << 16) | (e16[i] & 0xffu); }
};
inline HostView host_view(const ds_dag_batch* b) {
    return HostView{b->n_dags, b->node_off, b->edge_off, b->load_num, b->load_den, nullptr, nullptr, b->edges};
}
inline HostView host_view(const ds_dag_batch16* b) {
    return HostView{b->n_dags, b->node_off, b->edge_off, nullptr, nullptr, b->load, b->edges, nullptr};
}

// Packs `h` into ctx.small_in and points a's inputs at its device alias.
int small_inputs(const HostView& h, DeviceCtx& ctx, K1Args& a, cudaStream_t s) {
    const u64 n = h.n;
    const u32 nb = h.node_off[0], eb = h.edge_off[0];
    const u64 N = h.node_off[n] - nb, E = h.edge_off[n] - eb;
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t o_eo = al((n + 1) * 4), o_ln = al(o_eo + (n + 1) * 4), o_ld = al(o_ln + N * 8),
                 o_ed = al(o_ld + (h.ld ? N * 8 : 0)), bytes = o_ed + E * 4;
    if (int rc = ctx.small_in.ensure(bytes, true)) return rc;
    char* w = static_cast<char*>(ctx.small_in.p);
    const char* dv = static_cast<const char*>(ctx.small_in.dev);
    u32* no = reinterpret_cast<u32*>(w);
    u32* eo = reinterpret_cast<u32*>(w + o_eo);
    for (u64 i = 0; i <= n; ++i) {
        no[i] = h.node_off[i] - nb;
        eo[i] = h.edge_off[i] - eb;
    }
    int64_t* ln = reinterpret_cast<int64_t*>(w + o_ln);
    for (u64 i = 0; i < N; ++i) ln[i] = h.load(i);
    if (h.ld) std::memcpy(w + o_ld, h.ld, N * 8);
    u32* ed = reinterpret_cast<u32*>(w + o_ed);
    for (u64 i = 0; i < E; ++i) ed[i] = h.edge(i);
    // one H2D copy of the packed inputs into device memory, so the kernel's
    // dependent reads are not PCIe round trips (C1: kernel ~39 -> ~35 us,
    // raw ds_analyze_batch 41 -> 37 us); DS_SMALL_COPY=0: zero-copy reads
    static const bool copy = [] {
        const char* e = getenv("DS_SMALL_COPY");
        return !(e && e[0] == '0');
    }();
    if (copy) {
        if (int rc = ctx.small_dev.ensure(bytes)) return rc;
        DS_CUDA(cudaMemcpyAsync(ctx.small_dev.p, w, bytes, cudaMemcpyHostToDevice, s));
        dv = static_cast<const char*>(ctx.small_dev.p);
    }
    a.n_dags = n;
    a.node_off = reinterpret_cast<const u32*>(dv);
    a.edge_off = reinterpret_cast<const u32*>(dv + o_eo);
    a.load_num = reinterpret_cast<const u64*>(dv + o_ln);
    a.load_den = h.ld ? reinterpret_cast<const u64*>(dv + o_ld) : nullptr;
    a.edges = reinterpret_cast<const u32*>(dv + o_ed);
    return DS_OK;
}

int small_stream(int device, DeviceCtx& ctx, cudaStream_t& s) {
    DS_CUDA(cudaSetDevice(device));
    if (!ctx.init) {
        if (int rc = create_slot_streams(ctx)) return rc;
        ctx.init = true;
    }
    s = ctx.slot[0].s;
    return DS_OK;
}

// DS_SMALL_TRACE=1: the latency path's kernel time (CUDA events) on stderr
int small_launch_traced(const K1Args& a, bool detail, cudaStream_t s) {
    static const bool trace = [] {
        const char* e = getenv("DS_SMALL_TRACE");
        return e && e[0] == '1';
    }();
    if (!trace) {
        DS_CUDA(k1_small_launch(a, detail, s));
        return DS_OK;
    }
    cudaEvent_t e0, e1;
    DS_CUDA(cudaEventCreate(&e0));
    DS_CUDA(cudaEventCreate(&e1));
    DS_CUDA(cudaEventRecord(e0, s));
    DS_CUDA(k1_small_launch(a, detail, s));
    DS_CUDA(cudaEventRecord(e1, s));
    DS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    DS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    fprintf(stderr, "[small] k1_small<%d> %llu DAGs: %.1f us\n", int(detail), (unsigned long long)a.n_dags, 1e3 * ms);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return DS_OK;
}

// bounds mode (ds_analyze_batch / ds_analyze_batch16 for small host batches)
int analyze_small(const HostView& h, const PlatT<u64>& P, uint32_t mask, ds_results* out, int device) {
    K1Occupancy occ;
    if (int rc = configure(device, false, occ)) return rc;
    DeviceCtx& ctx = device_ctx(device);
    std::lock_guard<std::mutex> lock(ctx.mu);
    cudaStream_t s;
    if (int rc = small_stream(device, ctx, s)) return rc;
    K1Args a{};
    if (int rc = small_inputs(h, ctx, a, s)) return rc;
    const u64 n = h.n;
    const size_t o_b = 0, o_st = n * 80, o_ng = o_st + n * 4;
    if (int rc = ctx.small_out.ensure(o_ng + n * 2, true)) return rc;
    char* dv = static_cast<char*>(ctx.small_out.dev);
    a.plat = P;
    a.mask = mask;
    a.bounds = reinterpret_cast<int64_t*>(dv + o_b);
    a.status = reinterpret_cast<int32_t*>(dv + o_st);
    a.n_groups = reinterpret_cast<uint16_t*>(dv + o_ng);
    if (int rc = small_launch_traced(a, false, s)) return rc;
    DS_CUDA(cudaStreamSynchronize(s));
    const char* r = static_cast<const char*>(ctx.small_out.p);
    std::memcpy(out->bounds, r + o_b, n * 80);
    std::memcpy(out->status, r + o_st, n * 4);
    if (out->n_groups) std::memcpy(out->n_groups, r + o_ng, n * 2);
    return DS_OK;
}

// The bounds pass runs as k1_front + k1_back (K1Handoff) unless DS_K1_SPLIT=0
// selects the single-kernel variant (kept for A/B measurement and tests).
bool k1_split_enabled() {
    static const bool on = [] {
        const char* e = getenv("DS_K1_SPLIT");
        return !(e && e[0] == '0');
    }();
    return on;
}

int attach_handoff(K1Args& a, DevBuf& buf, u64 n_dags, u64 n_nodes) {
    a.h = K1Handoff{};
    if (!k1_split_enabled() || !(a.mask & DS_M_PROPOSED)) return DS_OK;
    if (int rc = buf.ensure(k1_handoff_bytes(n_dags, n_nodes))) return rc;
    a.h = k1_handoff_carve(buf.p, n_dags, n_nodes);
    return DS_OK;
}

// DAGs above 256 nodes: k1_big's tier queues and, above 512, its HBM warp
// states (allocated on first use, kept with the context's other scratch)
int attach_big(K1Args& a, DevBuf& q, DevBuf& scratch, u64 n_dags, u32 max_n) {
    a.big_q = nullptr;
    a.big_scratch = nullptr;
    if (max_n <= 256) return DS_OK;
    if (int rc = q.ensure(2 * n_dags * 4)) return rc;
    a.big_q = q.as<u32>();
    if (max_n > 512) {
        if (int rc = scratch.ensure(size_t(kBigGrid) * kBigScratchPerCta)) return rc;
        a.big_scratch = scratch.as<unsigned char>();
    }
    return DS_OK;
}

DeviceCtx& device_ctx(int dev) {
    static DeviceCtx ctx[64];
    return ctx[dev & 63];
}

constexpr u64 kChunk = 1ull << 14;  // smallest chunk worth a launch sequence
constexpr u64 kDefaultChunks = 5;  // 1M C5 DAGs e2e (round 2 kernels): 3 chunks 171 M/s, 4: 179, 5: 181, 6: 180, 8: 160;
                                    // after the k1_fast rework (tools/gpu_e2e_chunks.sh): 3: 210, 4: 219, 5: 229-232, 6: 230, 8: 221

// the second offset array of each wire form: edges, or adjacency words
inline const uint32_t* second_off(const ds_dag_batch* b) { return b->edge_off; }
inline const uint32_t* second_off(const ds_dag_batch16* b) { return b->edge_off; }
inline const uint32_t* second_off(const ds_dag_batch_tri* b) { return b->adj_off; }

int analyze_small_tri(const ds_dag_batch_tri* b, const PlatT<u64>& P, uint32_t mask, ds_results* out, int device);

template <class Batch>
int analyze_host(const Batch* b, const PlatT<u64>& P, uint32_t mask, ds_results* out, int device) {
    constexpr bool compact = std::is_same<Batch, ds_dag_batch16>::value;
    constexpr bool tri = std::is_same<Batch, ds_dag_batch_tri>::value;
    if constexpr (tri) {
        // (the size check of bigger batches runs per chunk, beside the GPU work)
        if (b->n_dags <= kSmallDags && small_enabled()) {
            if (batch_max_n(b->node_off, 0, b->n_dags) > 64)
                return fail(DS_EINVAL, "ds_dag_batch_tri: DAG with more than 64 nodes");
            return analyze_small_tri(b, P, mask, out, device);
        }
    } else {
        // the latency kernel covers DAGs up to 256 nodes; bigger ones take k1_big
        if (b->n_dags <= kSmallDags && small_enabled() && batch_max_n(b->node_off, 0, b->n_dags) <= 256)
            return analyze_small(host_view(b), P, mask, out, device);
    }
    DS_CUDA(cudaSetDevice(device));
    K1Occupancy occ;
    if (int rc = configure(device, false, occ)) return rc;
    DeviceCtx& ctx = device_ctx(device);
    std::lock_guard<std::mutex> lock(ctx.mu);
    if (!ctx.init) {
        if (int rc = create_slot_streams(ctx)) return rc;
        ctx.init = true;
    }
    const u64 n = b->n_dags;
    // a few equal chunks: enough to hide the copies behind the analysis, few
    // enough that every launch sequence fills the GPU (smaller first/last
    // chunks measured slower too). DS_CHUNKS=k overrides (tuning knob).
    static const std::vector<u64> weights = [] {
        // DS_CHUNK_WEIGHTS=a,b,c,... (relative chunk sizes) overrides both
        if (const char* w = getenv("DS_CHUNK_WEIGHTS")) {
            std::vector<u64> out;
            for (const char* p = w; *p;) {
                char* end = nullptr;
                const long v = strtol(p, &end, 10);
                if (end == p || v < 1) break;
                out.push_back(u64(v));
                p = *end == ',' ? end + 1 : end;
                if (!*end) break;
            }
            if (!out.empty() && out.size() <= 64) return out;
        }
        const char* e = getenv("DS_CHUNKS");
        const long v = e ? atol(e) : 0;
        return std::vector<u64>(size_t(v >= 1 && v <= 64 ? v : long(kDefaultChunks)), 1);
    }();
    u64 wsum = 0;
    for (u64 w : weights) wsum += w;
    std::vector<u64> bounds{0};
    for (u64 i = 0, acc = 0; i < weights.size(); ++i) {
        acc += weights[i];
        const u64 hi = std::min(n, (n * acc + wsum - 1) / wsum);
        if (hi - bounds.back() >= kChunk || (hi == n && hi > bounds.back())) bounds.push_back(hi);
    }
    if (bounds.back() != n) bounds.back() = n;  // small batches: one (or few) chunks
    if (bounds.size() == 1) bounds.push_back(n);
    // streams (and buffer sets) the chunks rotate over: one per chunk (up to
    // kMaxSlots), so no chunk waits for an earlier one's buffers and stream
    // priority follows chunk order; DS_STREAMS overrides
    static const int env_slots = [] {
        const char* e = getenv("DS_STREAMS");
        const int v = e ? atoi(e) : 0;
        return v >= 1 && v <= kMaxSlots ? v : 0;
    }();
    const int n_slots = env_slots ? env_slots : int(std::min<size_t>(bounds.size() - 1, kMaxSlots));
    // DS_E2E_TRACE=1: per-chunk event timeline on stderr (tuning aid)
    static const bool trace = [] {
        const char* e = getenv("DS_E2E_TRACE");
        return e && e[0] == '1';
    }();
    std::vector<cudaEvent_t> tev;
    auto tmark = [&](cudaStream_t st) -> int {
        if (!trace) return DS_OK;
        cudaEvent_t e;
        DS_CUDA(cudaEventCreate(&e));
        DS_CUDA(cudaEventRecord(e, st));
        tev.push_back(e);
        return DS_OK;
    };
    // DS_PIPE=0: each chunk's copies and kernels on its own slot stream
    // (chunks overlap as whole launch sequences). Default: four streams —
    // copy-in, front kernels (k1_fast .. k1_mid), back kernels (walk sort,
    // lane walks, retries), copy-out — chained by events, so chunk c's walks
    // run beside chunk c+1's front kernels and both directions of PCIe stay
    // busy.
    static const bool pipe = [] {
        const char* e = getenv("DS_PIPE");
        return !(e && e[0] == '0');
    }();
    static const int pipe_backs = [] {
        const char* e = getenv("DS_PIPE_BACKS");
        const int v = e ? atoi(e) : 2;
        return v >= 1 && v <= 3 ? v : 2;
    }();
    // DS_PIPE_SPLIT=0: front and back kernels on one stream (tuning knob)
    static const bool pipe_split = [] {
        const char* e = getenv("DS_PIPE_SPLIT");
        return !(e && e[0] == '0');
    }();
    if (pipe) {
        // a previous call that failed part-way may have left work in flight
        // on the slot buffers: drain it (free when the streams are idle)
        for (cudaStream_t st : ctx.pipe) DS_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < kMaxSlots; ++k) ctx.pev_live[k] = false;
    }
    const auto h0 = std::chrono::steady_clock::now();
    if (int rc = tmark(pipe ? ctx.pipe[0] : ctx.slot[0].s)) return rc;
    for (size_t c = 0; c + 1 < bounds.size(); ++c) {
        const u64 lo = bounds[c], hi = bounds[c + 1], nd = hi - lo;
        const int si = int(c % size_t(n_slots));
        Slot& sl = ctx.slot[si];
        cudaStream_t s_in = sl.s, s_front = sl.s, s_back = nullptr, s_out = sl.s;
        if (pipe) {
            s_in = ctx.pipe[0];
            s_front = ctx.pipe[1];
            // back streams in rotation: chunk c+1's lane walks fill the tail
            // of chunk c's (DS_PIPE_BACKS = 1..3 streams)
            static const int kBackStream[3] = {2, 4, 5};
            s_back = pipe_split ? ctx.pipe[kBackStream[c % size_t(pipe_backs)]] : ctx.pipe[1];
            s_out = ctx.pipe[3];
            // the slot's buffers are reused once its previous chunk's results left
            if (ctx.pev_live[si]) DS_CUDA(cudaEventSynchronize(ctx.pev[si][3]));
        }
        // indices are relative to node_off[0] / edge_off[0] (header contract)
        const uint32_t* eoff = second_off(b);
        const u64 n0 = b->node_off[lo] - b->node_off[0], n1 = b->node_off[hi] - b->node_off[0];
        const u64 e0 = eoff[lo] - eoff[0], e1 = eoff[hi] - eoff[0];  // tri: adjacency words
        const size_t nn = n1 - n0, ne = e1 - e0;
        if (!pipe) DS_CUDA(cudaStreamSynchronize(sl.s));  // the slot's buffers are reused
        if (int rc = sl.node_off.ensure((nd + 1) * 4)) return rc;
        if (int rc = sl.edge_off.ensure((nd + 1) * 4)) return rc;
        if (int rc = sl.ln.ensure(nn * 8)) return rc;
        if (int rc = sl.edges.ensure(tri ? ne * 32 * 4 : ne * 4)) return rc;  // tri: capacity, 32 edges per word
        bool has_den = false;
        if constexpr (!compact && !tri) has_den = b->load_den != nullptr;
        if (has_den) {
            if (int rc = sl.ldn.ensure(nn * 8)) return rc;
        }
        if (int rc = sl.status.ensure(nd * 4)) return rc;
        if (int rc = sl.bounds.ensure(nd * 80)) return rc;
        if (int rc = sl.ngroups.ensure(nd * 2)) return rc;
        if (int rc = sl.retry.ensure(2 * nd * 4)) return rc;  // two retry lists
        if (int rc = sl.retry_count.ensure(kK1Counters * 4)) return rc;
        DS_CUDA(cudaMemcpyAsync(sl.node_off.p, b->node_off + lo, (nd + 1) * 4, cudaMemcpyHostToDevice, s_in));
        if constexpr (tri) {
            if (int rc = sl.adj_off.ensure((nd + 1) * 4)) return rc;
            if (int rc = sl.ln16.ensure(nn * 2)) return rc;
            if (int rc = sl.adj.ensure(ne * 4)) return rc;
            if (int rc = sl.edge_cnt.ensure(nd * 4)) return rc;
            DS_CUDA(cudaMemcpyAsync(sl.adj_off.p, b->adj_off + lo, (nd + 1) * 4, cudaMemcpyHostToDevice, s_in));
            DS_CUDA(cudaMemcpyAsync(sl.ln16.p, b->load + n0, nn * 2, cudaMemcpyHostToDevice, s_in));
            DS_CUDA(cudaMemcpyAsync(sl.adj.p, b->adj + e0, ne * 4, cudaMemcpyHostToDevice, s_in));
        } else if constexpr (compact) {
            if (int rc = sl.ln16.ensure(nn * 2)) return rc;
            if (int rc = sl.edges16.ensure(ne * 2)) return rc;
            DS_CUDA(cudaMemcpyAsync(sl.edge_off.p, b->edge_off + lo, (nd + 1) * 4, cudaMemcpyHostToDevice, s_in));
            DS_CUDA(cudaMemcpyAsync(sl.ln16.p, b->load + n0, nn * 2, cudaMemcpyHostToDevice, s_in));
            DS_CUDA(cudaMemcpyAsync(sl.edges16.p, b->edges + e0, ne * 2, cudaMemcpyHostToDevice, s_in));
        } else {
            DS_CUDA(cudaMemcpyAsync(sl.edge_off.p, b->edge_off + lo, (nd + 1) * 4, cudaMemcpyHostToDevice, s_in));
            DS_CUDA(cudaMemcpyAsync(sl.ln.p, b->load_num + n0, nn * 8, cudaMemcpyHostToDevice, s_in));
            if (has_den) {
                DS_CUDA(cudaMemcpyAsync(sl.ldn.p, b->load_den + n0, nn * 8, cudaMemcpyHostToDevice, s_in));
            }
            DS_CUDA(cudaMemcpyAsync(sl.edges.p, b->edges + e0, ne * 4, cudaMemcpyHostToDevice, s_in));
        }
        if (pipe) {
            DS_CUDA(cudaEventRecord(ctx.pev[si][0], s_in));
            DS_CUDA(cudaStreamWaitEvent(s_front, ctx.pev[si][0], 0));
        }
        if (int rc = tmark(s_in)) return rc;
        // the 16-bit form widens on the device (the front stream); the
        // triangular one inside k1_launch (only what the general kernels take)
        if constexpr (compact) {
            k_widen16<<<296, 512, 0, s_front>>>(sl.ln16.as<const uint16_t>(), sl.edges16.as<const uint16_t>(), nn, ne,
                                                sl.ln.as<u64>(), sl.edges.as<u32>());
            DS_CUDA(cudaGetLastError());
        }
        K1Args a{};
        a.n_dags = nd;
        a.node_off = sl.node_off.as<const u32>();
        a.edge_off = sl.edge_off.as<const u32>();
        a.load_num = sl.ln.as<const u64>();
        a.load_den = has_den ? sl.ldn.as<const u64>() : nullptr;
        a.edges = sl.edges.as<const u32>();
        a.edge_cnt = tri ? sl.edge_cnt.as<const u32>() : nullptr;
        if constexpr (tri) {
            a.tri.adj = sl.adj.as<const u32>();
            a.tri.adj_off = sl.adj_off.as<const u32>();
            a.tri.ln16 = sl.ln16.as<const uint16_t>();
            a.tri.ln = sl.ln.as<u64>();
            a.tri.edge_off = sl.edge_off.as<u32>();
            a.tri.edge_cnt = sl.edge_cnt.as<u32>();
            a.tri.edges = sl.edges.as<u32>();
        }
        a.plat = P;
        a.mask = mask;
        a.status = sl.status.as<int32_t>();
        a.bounds = sl.bounds.as<int64_t>();
        a.n_groups = out->n_groups ? sl.ngroups.as<uint16_t>() : nullptr;
        a.retry = sl.retry.as<u32>();
        a.retry_count = sl.retry_count.as<u32>();
        a.retry2 = a.retry + nd;
        a.retry2_count = a.retry_count + 1;
        if (int rc = attach_handoff(a, sl.handoff, nd, nn)) return rc;
        const u32 max_n = batch_max_n(b->node_off, lo, hi);
        if (tri && max_n > 64) {  // nothing of this chunk is queued yet; drain the earlier ones
            for (cudaStream_t st : ctx.pipe) cudaStreamSynchronize(st);
            for (auto& slot : ctx.slot) cudaStreamSynchronize(slot.s);
            return fail(DS_EINVAL, "ds_dag_batch_tri: DAG with more than 64 nodes");
        }
        if (int rc = attach_big(a, sl.big_q, sl.big_scratch, nd, max_n)) return rc;
        DS_CUDA(k1_launch(a, occ, max_n, false, s_front, nullptr, pipe && pipe_split ? s_back : nullptr,
                          pipe && pipe_split ? ctx.pev[si][1] : nullptr));
        if (pipe) {
            DS_CUDA(cudaEventRecord(ctx.pev[si][2], s_back));
            DS_CUDA(cudaStreamWaitEvent(s_out, ctx.pev[si][2], 0));
        }
        if (int rc = tmark(s_out)) return rc;
        DS_CUDA(cudaMemcpyAsync(out->status + lo, sl.status.p, nd * 4, cudaMemcpyDeviceToHost, s_out));
        DS_CUDA(cudaMemcpyAsync(out->bounds + 10 * lo, sl.bounds.p, nd * 80, cudaMemcpyDeviceToHost, s_out));
        if (out->n_groups) {
            DS_CUDA(cudaMemcpyAsync(out->n_groups + lo, sl.ngroups.p, nd * 2, cudaMemcpyDeviceToHost, s_out));
        }
        if (pipe) {
            DS_CUDA(cudaEventRecord(ctx.pev[si][3], s_out));
            ctx.pev_live[si] = true;
        }
        if (int rc = tmark(s_out)) return rc;
    }
    const auto h1 = std::chrono::steady_clock::now();
    if (pipe) {
        DS_CUDA(cudaStreamSynchronize(ctx.pipe[3]));
    } else {
        for (auto& sl : ctx.slot) DS_CUDA(cudaStreamSynchronize(sl.s));
    }
    if (trace) {
        const auto h2 = std::chrono::steady_clock::now();
        auto us = [&](std::chrono::steady_clock::time_point t) {
            return std::chrono::duration<double, std::micro>(t - h0).count();
        };
        fprintf(stderr, "[e2e] host: enqueue done %.0f us, synchronised %.0f us\n", us(h1), us(h2));
        // per chunk: inputs landed, K1 done, results landed (ms from the start)
        for (size_t i = 1; i + 2 < tev.size(); i += 3) {
            float t[3];
            for (int k = 0; k < 3; ++k) DS_CUDA(cudaEventElapsedTime(&t[k], tev[0], tev[i + k]));
            fprintf(stderr, "[e2e] chunk %zu: h2d %.3f  k1 %.3f  d2h %.3f ms\n", i / 3, t[0], t[1], t[2]);
        }
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
    return DS_OK;
}

// ------------------------------------------------------------------ session
struct Session {
    int device = 0;
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    DevBuf node_off, edge_off, ln, ldn, edges, status, bounds, ngroups, retry, retry_count, handoff;
    K1Args args{};
    K1Occupancy occ;
    K1Marks marks;
    u32 max_n = 0;
    DevBuf big_q, big_scratch;
    u64 n_dags = 0;
    ~Session() {
        for (int i = 0; i < K1Marks::kMax; ++i)
            if (marks.ev[i]) cudaEventDestroy(marks.ev[i]);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (s) cudaStreamDestroy(s);
    }
};

// Upload a whole batch (rebased offsets) into fresh device buffers.
template <class Holder>
int upload(const ds_dag_batch* b, Holder& H, cudaStream_t s) {
    const u64 n = b->n_dags;
    const u32 nb = b->node_off[0], eb = b->edge_off[0];
    const u64 N = b->node_off[n] - nb, E = b->edge_off[n] - eb;
    std::vector<u32> no(n + 1), eo(n + 1);
    for (u64 i = 0; i <= n; ++i) {
        no[i] = b->node_off[i] - nb;
        eo[i] = b->edge_off[i] - eb;
    }
    if (int rc = H.node_off.ensure((n + 1) * 4)) return rc;
    if (int rc = H.edge_off.ensure((n + 1) * 4)) return rc;
    if (int rc = H.ln.ensure(N * 8)) return rc;
    if (int rc = H.ldn.ensure(N * 8)) return rc;
    if (int rc = H.edges.ensure(E * 4)) return rc;
    DS_CUDA(cudaMemcpyAsync(H.node_off.p, no.data(), (n + 1) * 4, cudaMemcpyHostToDevice, s));
    DS_CUDA(cudaMemcpyAsync(H.edge_off.p, eo.data(), (n + 1) * 4, cudaMemcpyHostToDevice, s));
    DS_CUDA(cudaMemcpyAsync(H.ln.p, b->load_num, N * 8, cudaMemcpyHostToDevice, s));
    if (b->load_den) DS_CUDA(cudaMemcpyAsync(H.ldn.p, b->load_den, N * 8, cudaMemcpyHostToDevice, s));
    DS_CUDA(cudaMemcpyAsync(H.edges.p, b->edges, E * 4, cudaMemcpyHostToDevice, s));
    DS_CUDA(cudaStreamSynchronize(s));
    return DS_OK;
}


}  // namespace ds

namespace ds {
// rank i of N owns DAGs [n*i/N, n*(i+1)/N) (paper_2602_20826_b200/shard.py)
inline u64 shard_lo(u64 n, int parts, int i) {
    return u64((unsigned __int128)n * u64(i) / u64(parts));
}

inline ds_dag_batch sub_batch(const ds_dag_batch* b, u64 lo, u64 hi) {
    ds_dag_batch sub = *b;
    const u64 nb = b->node_off[lo] - b->node_off[0], eb = b->edge_off[lo] - b->edge_off[0];
    sub.n_dags = hi - lo;
    sub.node_off = b->node_off + lo;
    sub.edge_off = b->edge_off + lo;
    sub.load_num = b->load_num + nb;
    sub.load_den = b->load_den ? b->load_den + nb : nullptr;
    sub.edges = b->edges + eb;
    return sub;
}

inline ds_dag_batch16 sub_batch(const ds_dag_batch16* b, u64 lo, u64 hi) {
    ds_dag_batch16 sub = *b;
    sub.n_dags = hi - lo;
    sub.node_off = b->node_off + lo;
    sub.edge_off = b->edge_off + lo;
    sub.load = b->load + (b->node_off[lo] - b->node_off[0]);
    sub.edges = b->edges + (b->edge_off[lo] - b->edge_off[0]);
    return sub;
}

inline ds_dag_batch_tri sub_batch(const ds_dag_batch_tri* b, u64 lo, u64 hi) {
    ds_dag_batch_tri sub = *b;
    sub.n_dags = hi - lo;
    sub.node_off = b->node_off + lo;
    sub.adj_off = b->adj_off + lo;
    sub.load = b->load + (b->node_off[lo] - b->node_off[0]);
    sub.adj = b->adj + (b->adj_off[lo] - b->adj_off[0]);
    return sub;
}

int analyze_one(const ds_dag_batch* b, const ds_platform* p, uint32_t mask, ds_results* r, int dev);
int analyze_one(const ds_dag_batch16* b, const ds_platform* p, uint32_t mask, ds_results* r, int dev);
int analyze_one(const ds_dag_batch_tri* b, const ds_platform* p, uint32_t mask, ds_results* r, int dev);

// contiguous shards over devices, one host thread per device, no collective
// (DAGs are independent, experiment.cpp:56-57); results land in DAG order
template <class Batch>
int analyze_multi(const Batch* batch, const ds_platform* platform, uint32_t method_mask, ds_results* out,
                  const int* devices, int n_devices) {
    if (!batch || !out || !devices || n_devices < 1) return fail(DS_EINVAL, "bad arguments");
    const u64 n = batch->n_dags;
    std::vector<int> rcs(n_devices, DS_OK);
    std::vector<std::string> errs(n_devices);
    std::vector<std::thread> th;
    for (int i = 0; i < n_devices; ++i) {
        const u64 lo = shard_lo(n, n_devices, i), hi = shard_lo(n, n_devices, i + 1);
        th.emplace_back([&, i, lo, hi] {
            const Batch sub = sub_batch(batch, lo, hi);  // shifted pointers (relative-index contract)
            ds_results r = *out;
            r.status = out->status + lo;
            r.bounds = out->bounds + 10 * lo;
            r.n_groups = out->n_groups ? out->n_groups + lo : nullptr;
            rcs[i] = analyze_one(&sub, platform, method_mask, &r, devices[i]);
            errs[i] = g_err;
        });
    }
    for (auto& t : th) t.join();
    for (int i = 0; i < n_devices; ++i) {
        if (rcs[i] != DS_OK) return fail(rcs[i], errs[i]);
    }
    return DS_OK;
}
}  // namespace ds

using namespace ds;

extern "C" {

const char* ds_last_error(void) { return g_err.c_str(); }
const char* ds_version(void) { return "dagsched_b200 0.2 (sm_100a)"; }

int ds_pinned_alloc(size_t bytes, void** out) {
    if (!out) return fail(DS_EINVAL, "NULL output pointer");
    *out = nullptr;
    DS_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
    return DS_OK;
}

int ds_pinned_free(void* p) {
    if (p) DS_CUDA(cudaFreeHost(p));
    return DS_OK;
}

int ds_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(DS_ENODEV, cudaGetErrorString(e));
    }
    *count = c;
    return DS_OK;
}

int ds_analyze_batch16(const ds_dag_batch16* batch, const ds_platform* platform, uint32_t method_mask,
                       ds_results* out, int device) {
    if (!batch || !out || !out->status || !out->bounds) return fail(DS_EINVAL, "NULL batch or results");
    PlatT<u64> P;
    if (int rc = check_platform(platform, P)) return rc;
    if (batch->n_dags == 0) return DS_OK;
    if (!batch->node_off || !batch->edge_off || !batch->load || !batch->edges) return fail(DS_EINVAL, "NULL array");
    return analyze_host(batch, P, method_mask & DS_M_ALL, out, device);
}

int ds_analyze_batch_tri(const ds_dag_batch_tri* batch, const ds_platform* platform, uint32_t method_mask,
                         ds_results* out, int device) {
    if (!batch || !out || !out->status || !out->bounds) return fail(DS_EINVAL, "NULL batch or results");
    PlatT<u64> P;
    if (int rc = check_platform(platform, P)) return rc;
    if (batch->n_dags == 0) return DS_OK;
    if (!batch->node_off || !batch->adj_off || !batch->load || !batch->adj) return fail(DS_EINVAL, "NULL array");
    return analyze_host(batch, P, method_mask & DS_M_ALL, out, device);
}

int ds_analyze_batch(const ds_dag_batch* batch, const ds_platform* platform, uint32_t method_mask,
                     ds_results* out, int device, void* stream, uint32_t flags) {
    if (!batch || !out || !out->status || !out->bounds) return fail(DS_EINVAL, "NULL batch or results");
    PlatT<u64> P;
    if (int rc = check_platform(platform, P)) return rc;
    if (batch->n_dags == 0) return DS_OK;
    if (!(flags & DS_F_DEVICE_PTRS)) return analyze_host(batch, P, method_mask & DS_M_ALL, out, device);
    DS_CUDA(cudaSetDevice(device));
    K1Occupancy occ;
    if (int rc = configure(device, false, occ)) return rc;
    DeviceCtx& ctx = device_ctx(device);
    std::lock_guard<std::mutex> lock(ctx.mu);
    if (int rc = ctx.retry.ensure(2 * batch->n_dags * 4)) return rc;
    if (int rc = ctx.retry_count.ensure(kK1Counters * 4)) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    u32 ends[2];  // node_off[0], node_off[n]: sizes the split pass's scratch
    DS_CUDA(cudaMemcpyAsync(&ends[0], batch->node_off, 4, cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaMemcpyAsync(&ends[1], batch->node_off + batch->n_dags, 4, cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaStreamSynchronize(s));
    K1Args a{};
    a.n_dags = batch->n_dags;
    a.node_off = batch->node_off;
    a.edge_off = batch->edge_off;
    a.load_num = reinterpret_cast<const u64*>(batch->load_num);
    a.load_den = reinterpret_cast<const u64*>(batch->load_den);
    a.edges = batch->edges;
    a.plat = P;
    a.mask = method_mask & DS_M_ALL;
    a.status = out->status;
    a.bounds = out->bounds;
    a.n_groups = out->n_groups;
    a.retry = ctx.retry.as<u32>();
    a.retry_count = ctx.retry_count.as<u32>();
    a.retry2 = a.retry + batch->n_dags;
    a.retry2_count = a.retry_count + 1;
    if (int rc = attach_handoff(a, ctx.handoff, batch->n_dags, u64(ends[1] - ends[0]))) return rc;
    // device pointers: size classes are unknown on the host, so every
    // size-class kernel runs (each skips the DAGs of other classes after two
    // offset loads)
    if (int rc = attach_big(a, ctx.big_q, ctx.big_scratch, batch->n_dags, DS_MAX_NODES)) return rc;
    DS_CUDA(k1_launch(a, occ, DS_MAX_NODES, false, s));
    // the scratch is reused by the next call: finish before releasing it
    DS_CUDA(cudaStreamSynchronize(s));
    return DS_OK;
}

int ds_shard_range(uint64_t n_dags, int n_shards, int shard, uint64_t* lo, uint64_t* hi) {
    if (n_shards < 1 || shard < 0 || shard >= n_shards || !lo || !hi) return fail(DS_EINVAL, "bad shard");
    *lo = shard_lo(n_dags, n_shards, shard);
    *hi = shard_lo(n_dags, n_shards, shard + 1);
    return DS_OK;
}

int ds_analyze_batch_multi(const ds_dag_batch* batch, const ds_platform* platform, uint32_t method_mask,
                           ds_results* out, const int* devices, int n_devices) {
    return analyze_multi(batch, platform, method_mask, out, devices, n_devices);
}

int ds_analyze_batch16_multi(const ds_dag_batch16* batch, const ds_platform* platform, uint32_t method_mask,
                             ds_results* out, const int* devices, int n_devices) {
    return analyze_multi(batch, platform, method_mask, out, devices, n_devices);
}

int ds_analyze_batch_tri_multi(const ds_dag_batch_tri* batch, const ds_platform* platform, uint32_t method_mask,
                               ds_results* out, const int* devices, int n_devices) {
    return analyze_multi(batch, platform, method_mask, out, devices, n_devices);
}

}  // extern "C"

namespace ds {
int analyze_one(const ds_dag_batch* b, const ds_platform* p, uint32_t mask, ds_results* r, int dev) {
    return ds_analyze_batch(b, p, mask, r, dev, nullptr, 0);
}
int analyze_one(const ds_dag_batch16* b, const ds_platform* p, uint32_t mask, ds_results* r, int dev) {
    return ds_analyze_batch16(b, p, mask, r, dev);
}
int analyze_one(const ds_dag_batch_tri* b, const ds_platform* p, uint32_t mask, ds_results* r, int dev) {
    return ds_analyze_batch_tri(b, p, mask, r, dev);
}
// a small triangular batch: expanded to the wide form on the host, then the
// latency path
int analyze_small_tri(const ds_dag_batch_tri* b, const PlatT<u64>& P, uint32_t mask, ds_results* out, int device) {
    const u64 n = b->n_dags;
    std::vector<uint32_t> no(n + 1), eo(n + 1, 0), ed;
    std::vector<int64_t> ln;
    const u32 nb = b->node_off[0], ab = b->adj_off[0];
    for (u64 d = 0; d < n; ++d) {
        no[d] = b->node_off[d] - nb;
        const int nn = int(b->node_off[d + 1] - b->node_off[d]);
        const u32* w = b->adj + (b->adj_off[d] - ab);
        const u32 nw = b->adj_off[d + 1] - b->adj_off[d];
        for (int v = 0; v < nn; ++v) ln.push_back(b->load[no[d] + v]);
        for (int u = 0; u < nn; ++u)  // (from, to) order
            for (int v = u + 1; v < nn; ++v) {
                const u32 bit = u32(v) * u32(v - 1) / 2 + u32(u);
                if ((bit >> 5) < nw && ((w[bit >> 5] >> (bit & 31)) & 1)) ed.push_back((u32(u) << 16) | u32(v));
            }
        eo[d + 1] = u32(ed.size());
    }
    no[n] = b->node_off[n] - nb;
    const ds_dag_batch wide{n, no.data(), eo.data(), ln.data(), nullptr, ed.data()};
    return analyze_small(host_view(&wide), P, mask, out, device);
}
// schedule-detail mode for a small host batch: one k1_small launch over
// mapped buffers (see analyze_small)
int schedule_small(const ds_dag_batch* b, const PlatT<u64>& P, ds_scheme_out* out, int device, DeviceCtx& ctx) {
    K1Occupancy occ;
    if (int rc = configure(device, true, occ)) return rc;
    std::lock_guard<std::mutex> lock(ctx.mu);
    cudaStream_t s;
    if (int rc = small_stream(device, ctx, s)) return rc;
    K1Args a{};
    const HostView h = host_view(b);
    if (int rc = small_inputs(h, ctx, a, s)) return rc;
    const u64 n = h.n, N = b->node_off[n] - b->node_off[0];
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t o_ent = 0, o_grp = al(o_ent + 2 * N * sizeof(ds_entity_rec)), o_b = al(o_grp + N * sizeof(ds_group_rec)),
                 o_st = al(o_b + n * 80), o_ne = al(o_st + n * 4), o_ng = al(o_ne + n * 2), o_nd = al(o_ng + n * 2),
                 o_nb = al(o_nd + n * 2), o_ndg = al(o_nb + N * 2), o_ub = al(o_ndg + N * 2), o_unl = al(o_ub + n * 8);
    const u64 unl_words = unl_layout(b->node_off, n, nullptr);
    const size_t bytes = o_unl + unl_words * 8;
    if (int rc = ctx.small_out.ensure(bytes, true)) return rc;
    char* dv = static_cast<char*>(ctx.small_out.dev);
    a.plat = P;
    a.mask = DS_M_ALL;
    a.det.entities = reinterpret_cast<ds_entity_rec*>(dv + o_ent);
    a.det.groups = reinterpret_cast<ds_group_rec*>(dv + o_grp);
    a.det.bounds = reinterpret_cast<int64_t*>(dv + o_b);
    a.det.status = reinterpret_cast<int32_t*>(dv + o_st);
    a.det.n_entities = reinterpret_cast<uint16_t*>(dv + o_ne);
    a.det.n_groups = reinterpret_cast<uint16_t*>(dv + o_ng);
    a.det.n_div_groups = reinterpret_cast<uint16_t*>(dv + o_nd);
    a.det.node_block = reinterpret_cast<int16_t*>(dv + o_nb);
    a.det.node_div_group = reinterpret_cast<int16_t*>(dv + o_ndg);
    a.det.unlaunched = reinterpret_cast<uint64_t*>(dv + o_unl);
    unl_layout(b->node_off, n, reinterpret_cast<u64*>(static_cast<char*>(ctx.small_out.p) + o_ub));
    a.unl_base = reinterpret_cast<const u64*>(dv + o_ub);
    if (int rc = small_launch_traced(a, true, s)) return rc;
    DS_CUDA(cudaStreamSynchronize(s));
    const char* r = static_cast<const char*>(ctx.small_out.p);
    auto put = [&](void* dst, size_t off, size_t len) {
        if (dst) std::memcpy(dst, r + off, len);
    };
    put(out->status, o_st, n * 4);
    put(out->n_entities, o_ne, n * 2);
    put(out->n_groups, o_ng, n * 2);
    put(out->n_div_groups, o_nd, n * 2);
    put(out->node_block, o_nb, N * 2);
    put(out->node_div_group, o_ndg, N * 2);
    put(out->entities, o_ent, 2 * N * sizeof(ds_entity_rec));
    put(out->groups, o_grp, N * sizeof(ds_group_rec));
    put(out->bounds, o_b, n * 80);
    put(out->unlaunched, o_unl, unl_words * 8);
    return DS_OK;
}

// K1 in detail mode over a host batch; results stay in the device context's
// out arena (ctx.det.v). The caller holds ctx.mu and the stream slot 0.
int run_detail(const ds_dag_batch* b, const PlatT<u64>& P, int device, DeviceCtx& ctx) {
    const u64 n = b->n_dags;
    DS_CUDA(cudaSetDevice(device));
    K1Occupancy occ;
    if (int rc = configure(device, true, occ)) return rc;
    if (!ctx.init) {
        if (int rc = create_slot_streams(ctx)) return rc;
        ctx.init = true;
    }
    cudaStream_t s = ctx.slot[0].s;
    DetailCtx& D = ctx.det;
    DetailView& v = D.v;
    const u32 nb0 = b->node_off[0], eb0 = b->edge_off[0];
    const u64 N = b->node_off[n] - nb0, E = b->edge_off[n] - eb0;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    // ---- inputs: rebased offsets, loads, edges in one pinned stage -> one H2D
    const size_t i_no = 0, i_eo = al(i_no + (n + 1) * 4), i_ln = al(i_eo + (n + 1) * 4), i_ld = al(i_ln + N * 8),
                 i_ed = al(i_ld + (b->load_den ? N * 8 : 0)), i_ub = al(i_ed + E * 4), in_bytes = al(i_ub + n * 8);
    if (int rc = D.in_stage.ensure(in_bytes)) return rc;
    if (int rc = D.in.ensure(in_bytes)) return rc;
    char* st = static_cast<char*>(D.in_stage.p);
    u32* no = reinterpret_cast<u32*>(st + i_no);
    u32* eo = reinterpret_cast<u32*>(st + i_eo);
    for (u64 i = 0; i <= n; ++i) {
        no[i] = b->node_off[i] - nb0;
        eo[i] = b->edge_off[i] - eb0;
    }
    std::memcpy(st + i_ln, b->load_num, N * 8);
    if (b->load_den) std::memcpy(st + i_ld, b->load_den, N * 8);
    std::memcpy(st + i_ed, b->edges, E * 4);
    v.unl_words = unl_layout(b->node_off, n, reinterpret_cast<u64*>(st + i_ub));
    DS_CUDA(cudaMemcpyAsync(D.in.p, st, in_bytes, cudaMemcpyHostToDevice, s));
    char* di = static_cast<char*>(D.in.p);
    v.node_off = reinterpret_cast<u32*>(di + i_no);
    v.edge_off = reinterpret_cast<u32*>(di + i_eo);
    v.ln = reinterpret_cast<u64*>(di + i_ln);
    v.ldn = b->load_den ? reinterpret_cast<u64*>(di + i_ld) : nullptr;
    v.edges = reinterpret_cast<u32*>(di + i_ed);
    // ---- outputs: one arena; node_block/node_div_group (0xff) and entity /
    // group records (0) are adjacent so two memsets initialise them
    v.o_nb = 0;
    v.o_ndg = v.o_nb + N * 2;
    v.o_ent = al(v.o_ndg + N * 2);
    v.o_grp = v.o_ent + 2 * N * sizeof(ds_entity_rec);
    v.o_status = al(v.o_grp + N * sizeof(ds_group_rec));
    v.o_ne = al(v.o_status + n * 4);
    v.o_ng = al(v.o_ne + n * 2);
    v.o_nd = al(v.o_ng + n * 2);
    v.o_bounds = al(v.o_nd + n * 2);
    v.o_unl = al(v.o_bounds + n * 80);
    v.out_bytes = al(v.o_unl + v.unl_words * 8);
    if (int rc = D.out.ensure(v.out_bytes)) return rc;
    if (int rc = D.retry.ensure(2 * n * 4)) return rc;
    if (int rc = D.retry_count.ensure(kK1Counters * 4)) return rc;
    char* dout = static_cast<char*>(D.out.p);
    v.nb = reinterpret_cast<int16_t*>(dout + v.o_nb);
    v.ndg = reinterpret_cast<int16_t*>(dout + v.o_ndg);
    v.ent = reinterpret_cast<ds_entity_rec*>(dout + v.o_ent);
    v.grp = reinterpret_cast<ds_group_rec*>(dout + v.o_grp);
    v.status = reinterpret_cast<int32_t*>(dout + v.o_status);
    v.ne = reinterpret_cast<uint16_t*>(dout + v.o_ne);
    v.ng = reinterpret_cast<uint16_t*>(dout + v.o_ng);
    v.nd = reinterpret_cast<uint16_t*>(dout + v.o_nd);
    v.bounds = reinterpret_cast<int64_t*>(dout + v.o_bounds);
    v.unl = reinterpret_cast<uint64_t*>(dout + v.o_unl);
    DS_CUDA(cudaMemsetAsync(dout + v.o_nb, 0xff, N * 4, s));
    DS_CUDA(cudaMemsetAsync(dout + v.o_ent, 0, v.o_status - v.o_ent, s));
    K1Args a{};
    a.n_dags = n;
    a.node_off = v.node_off;
    a.edge_off = v.edge_off;
    a.load_num = v.ln;
    a.load_den = v.ldn;
    a.edges = v.edges;
    a.plat = P;
    a.mask = DS_M_ALL;
    a.det.status = v.status;
    a.det.n_entities = v.ne;
    a.det.n_groups = v.ng;
    a.det.n_div_groups = v.nd;
    a.det.node_block = v.nb;
    a.det.node_div_group = v.ndg;
    a.det.entities = v.ent;
    a.det.groups = v.grp;
    a.det.bounds = v.bounds;
    a.det.unlaunched = v.unl;
    a.unl_base = reinterpret_cast<const u64*>(di + i_ub);
    a.retry = D.retry.as<u32>();
    a.retry_count = D.retry_count.as<u32>();
    a.retry2 = a.retry + n;
    a.retry2_count = a.retry_count + 1;
    const u32 max_n = batch_max_n(b->node_off, 0, n);
    if (int rc = attach_big(a, D.big_q, D.big_scratch, n, max_n)) return rc;
    DS_CUDA(k1_launch(a, occ, max_n, true, s));
    return DS_OK;
}
}  // namespace ds

extern "C" {

int ds_schedule_batch(const ds_dag_batch* b, const ds_platform* platform, ds_scheme_out* out, int device) {
    if (!b || !out) return fail(DS_EINVAL, "NULL batch or output");
    PlatT<u64> P;
    if (int rc = check_platform(platform, P)) return rc;
    const u64 n = b->n_dags;
    if (n == 0) return DS_OK;
    DeviceCtx& ctx = device_ctx(device);
    if (n <= kSmallDags && small_enabled() && batch_max_n(b->node_off, 0, n) <= 256)
        return schedule_small(b, P, out, device, ctx);
    std::lock_guard<std::mutex> lock(ctx.mu);
    if (int rc = run_detail(b, P, device, ctx)) return rc;
    DetailCtx& D = ctx.det;
    const DetailView& v = D.v;
    cudaStream_t s = ctx.slot[0].s;
    // one D2H of the whole out arena, then host copies into the caller's arrays
    if (int rc = D.out_stage.ensure(v.out_bytes)) return rc;
    DS_CUDA(cudaMemcpyAsync(D.out_stage.p, D.out.p, v.out_bytes, cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaStreamSynchronize(s));
    const char* h = static_cast<const char*>(D.out_stage.p);
    const u64 N = b->node_off[n] - b->node_off[0];
    auto put = [&](void* dst, size_t off, size_t bytes) {
        if (dst) std::memcpy(dst, h + off, bytes);
    };
    put(out->status, v.o_status, n * 4);
    put(out->n_entities, v.o_ne, n * 2);
    put(out->n_groups, v.o_ng, n * 2);
    put(out->n_div_groups, v.o_nd, n * 2);
    put(out->node_block, v.o_nb, N * 2);
    put(out->node_div_group, v.o_ndg, N * 2);
    put(out->entities, v.o_ent, 2 * N * sizeof(ds_entity_rec));
    put(out->groups, v.o_grp, N * sizeof(ds_group_rec));
    put(out->bounds, v.o_bounds, n * 80);
    put(out->unlaunched, v.o_unl, v.unl_words * 8);
    return DS_OK;
}

int ds_validate_batch(const ds_dag_batch* b, const ds_platform* platform, int samples, int64_t smin_num,
                      int64_t smin_den, int64_t smax_num, int64_t smax_den, uint64_t seed, int32_t* status,
                      int32_t* violations, double* tight_worst, double* tight_scaled, ds_validation* summary,
                      int device) {
    if (!b || samples < 0) return fail(DS_EINVAL, "bad arguments");
    PlatT<u64> P;
    if (int rc = check_platform(platform, P)) return rc;
    // FactorSource (simulator.cpp:18-30): 0 < min <= max <= 1 on a 1/1024 grid
    long long lo = 1024, hi = 1024;
    if (samples > 0) {
        if (smin_den <= 0 || smax_den <= 0 || smin_num <= 0 || smax_num > smax_den ||
            (__int128)smin_num * smax_den > (__int128)smax_num * smin_den)
            return fail(DS_EINVAL, "scale factors must satisfy 0 < min <= max <= 1");
        lo = std::max(1LL, (long long)((smin_num * 1024 + smin_den - 1) / smin_den));  // ceil
        hi = std::max(lo, (long long)(smax_num * 1024 / smax_den));                  // floor
    }
    const u64 n = b->n_dags;
    if (n == 0) return DS_OK;
    DeviceCtx& ctx = device_ctx(device);
    std::lock_guard<std::mutex> lock(ctx.mu);
    if (int rc = run_detail(b, P, device, ctx)) return rc;
    DetailCtx& D = ctx.det;
    const DetailView& v = D.v;
    cudaStream_t s = ctx.slot[0].s;
    const u64 per = u64(samples) + 1, T = n * per;
    if (int rc = D.k4_over.ensure(T)) return rc;
    if (int rc = D.k4_ratio.ensure(T * 8)) return rc;
    if (int rc = D.k4_st.ensure(T * 4)) return rc;
    k4_launch(n, v.node_off, v.status, v.ng, v.grp, v.ent, v.bounds, samples, lo, hi, seed,
              D.k4_over.as<unsigned char>(), D.k4_ratio.as<double>(), D.k4_st.as<int32_t>(), s);
    DS_CUDA(cudaGetLastError());
    std::vector<unsigned char> h_over(T);
    std::vector<double> h_ratio(T);
    std::vector<int32_t> h_st(T);
    DS_CUDA(cudaMemcpyAsync(h_over.data(), D.k4_over.p, T, cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaMemcpyAsync(h_ratio.data(), D.k4_ratio.p, T * 8, cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaMemcpyAsync(h_st.data(), D.k4_st.p, T * 4, cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaStreamSynchronize(s));
    // experiment.cpp:179-239 reductions, in the same order (samples, then tasks)
    ds_validation sum{int64_t(n), int64_t(n * per), 0, 0.0, 0.0};
    double worst_sum = 0.0, scaled_total = 0.0;
    for (u64 d = 0; d < n; ++d) {
        int sd = DS_OK;
        for (u64 k = 0; k < per; ++k) sd = sd != DS_OK ? sd : h_st[d * per + k];
        int viol = 0;
        double scaled = 0.0;
        for (int s = 0; s < samples; ++s) {
            viol += h_over[d * per + s];
            scaled += h_ratio[d * per + s];
        }
        viol += h_over[d * per + samples];
        const double tw = h_ratio[d * per + samples];
        const double ts = samples > 0 ? scaled / samples : 0.0;
        if (status) status[d] = sd;
        if (violations) violations[d] = viol;
        if (tight_worst) tight_worst[d] = tw;
        if (tight_scaled) tight_scaled[d] = ts;
        sum.violations += viol;
        worst_sum += tw;
        scaled_total += ts;
    }
    sum.mean_tightness_worst = worst_sum / double(n);
    sum.mean_tightness_scaled = scaled_total / double(n);
    if (summary) *summary = sum;
    return DS_OK;
}

int ds_session_create(const ds_dag_batch* b, const ds_platform* platform, uint32_t method_mask, int device,
                      void** session) {
    if (!b || !session) return fail(DS_EINVAL, "NULL argument");
    PlatT<u64> P;
    if (int rc = check_platform(platform, P)) return rc;
    auto* S = new Session();
    S->device = device;
    S->n_dags = b->n_dags;
    auto bail = [&](int rc) {
        delete S;
        return rc;
    };
    if (cudaSetDevice(device) != cudaSuccess) return bail(fail(DS_ECUDA, "cudaSetDevice"));
    if (int rc = configure(device, false, S->occ)) return bail(rc);
    for (int i = 0; i < K1Marks::kMax; ++i) S->marks.ev[i] = nullptr;
    if (cudaStreamCreateWithFlags(&S->s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&S->e0) != cudaSuccess || cudaEventCreate(&S->e1) != cudaSuccess) {
        return bail(fail(DS_ECUDA, "stream/event creation failed"));
    }
    for (int i = 0; i < K1Marks::kMax; ++i) {
        if (cudaEventCreate(&S->marks.ev[i]) != cudaSuccess) return bail(fail(DS_ECUDA, "event creation failed"));
    }
    if (int rc = upload(b, *S, S->s)) return bail(rc);
    const u64 n = b->n_dags;
    S->max_n = batch_max_n(b->node_off, 0, n);
    int rc = DS_OK;
    rc = rc ? rc : S->status.ensure(n * 4);
    rc = rc ? rc : S->bounds.ensure(n * 80);
    rc = rc ? rc : S->ngroups.ensure(n * 2);
    rc = rc ? rc : S->retry.ensure(2 * n * 4);
    rc = rc ? rc : S->retry_count.ensure(kK1Counters * 4);
    if (rc) return bail(rc);
    K1Args& a = S->args;
    a.n_dags = n;
    a.node_off = S->node_off.as<const u32>();
    a.edge_off = S->edge_off.as<const u32>();
    a.load_num = S->ln.as<const u64>();
    a.load_den = b->load_den ? S->ldn.as<const u64>() : nullptr;
    a.edges = S->edges.as<const u32>();
    a.plat = P;
    a.mask = method_mask & DS_M_ALL;
    a.status = S->status.as<int32_t>();
    a.bounds = S->bounds.as<int64_t>();
    a.n_groups = S->ngroups.as<uint16_t>();
    a.retry = S->retry.as<u32>();
    a.retry_count = S->retry_count.as<u32>();
    a.retry2 = a.retry + n;
    a.retry2_count = a.retry_count + 1;
    if (int rc2 = attach_handoff(a, S->handoff, n, u64(b->node_off[n] - b->node_off[0]))) return bail(rc2);
    if (int rc2 = attach_big(a, S->big_q, S->big_scratch, n, S->max_n)) return bail(rc2);
    *session = S;
    return DS_OK;
}

int ds_session_run(void* session, float* kernel_ms) {
    auto* S = static_cast<Session*>(session);
    DS_CUDA(cudaSetDevice(S->device));
    DS_CUDA(cudaEventRecord(S->e0, S->s));
    DS_CUDA(k1_launch(S->args, S->occ, S->max_n, false, S->s, &S->marks));
    DS_CUDA(cudaEventRecord(S->e1, S->s));
    DS_CUDA(cudaEventSynchronize(S->e1));
    if (kernel_ms) DS_CUDA(cudaEventElapsedTime(kernel_ms, S->e0, S->e1));
    return DS_OK;
}

int ds_session_kernel_times(void* session, float* ms, const char** names, int max) {
    auto* S = static_cast<Session*>(session);
    if (!S || max < 0) return -fail(DS_EINVAL, "bad argument");
    const K1Marks& m = S->marks;
    int k = 0;
    for (int i = 0; i < m.n && k < max; ++i, ++k) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, i == 0 ? S->e0 : m.ev[i - 1], m.ev[i]) != cudaSuccess)
            return -fail(DS_ECUDA, "cudaEventElapsedTime");
        if (ms) ms[k] = t;
        if (names) names[k] = m.name[i];
    }
    return k;
}

int ds_session_results(void* session, ds_results* out) {
    auto* S = static_cast<Session*>(session);
    DS_CUDA(cudaSetDevice(S->device));
    DS_CUDA(cudaStreamSynchronize(S->s));
    const u64 n = S->n_dags;
    if (out->status) DS_CUDA(cudaMemcpy(out->status, S->status.p, n * 4, cudaMemcpyDeviceToHost));
    if (out->bounds) DS_CUDA(cudaMemcpy(out->bounds, S->bounds.p, n * 80, cudaMemcpyDeviceToHost));
    if (out->n_groups) DS_CUDA(cudaMemcpy(out->n_groups, S->ngroups.p, n * 2, cudaMemcpyDeviceToHost));
    return DS_OK;
}

int ds_session_free(void* session) {
    auto* S = static_cast<Session*>(session);
    if (!S) return DS_OK;
    cudaSetDevice(S->device);
    if (S->s) cudaStreamSynchronize(S->s);
    delete S;  // ~Session releases the stream and events
    return DS_OK;
}

}  // extern "C"

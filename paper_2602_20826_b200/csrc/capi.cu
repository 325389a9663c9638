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
#include "k1_analysis.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace ds {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define DS_CUDA(call)                                                                           \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess) return fail(DS_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

int check_platform(const ds_platform* p, Plat& out) {
    if (!p) return fail(DS_EINVAL, "platform is NULL");
    if (p->sm_count < 1) return fail(DS_EINVAL, "sm_count must be >= 1");
    long long n = p->tmin_num, d = p->tmin_den;
    if (d == 0) return fail(DS_EINVAL, "t_min denominator is zero");
    if (d < 0) {
        n = -n;
        d = -d;
    }
    if (n <= 0) return fail(DS_EINVAL, "t_min must be positive");
    u64 g = 1, a = u64(n), b = u64(d);
    while (b) {
        u64 t = a % b;
        a = b;
        b = t;
    }
    g = a;
    out.M = p->sm_count;
    out.tmin = Rat{u64(n) / g, u64(d) / g};
    return DS_OK;
}

// ------------------------------------------------------------ kernel launch
constexpr int kWarpsSmall = 4;  // WarpState<1> per warp, 4 warps per CTA
constexpr int kWarpsBig = 1;    // WarpState<4> (n <= 256) is ~66 KB

template <int W, bool DETAIL>
size_t smem_bytes(int warps) {
    return sizeof(WarpState<W>) * size_t(warps);
}

struct LaunchCfg {
    int grid_small = 0, grid_big = 0;
};

template <bool DETAIL>
int configure(int device, LaunchCfg& cfg) {
    static std::mutex mu;
    static LaunchCfg cache[64];
    static bool ready[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    const int slot = device * 2 + (DETAIL ? 1 : 0);
    if (slot < 64 && ready[slot]) {
        cfg = cache[slot];
        return DS_OK;
    }
    int sms = 0;
    DS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const size_t s1 = smem_bytes<1, DETAIL>(kWarpsSmall), s4 = smem_bytes<4, DETAIL>(kWarpsBig);
    DS_CUDA(cudaFuncSetAttribute(k1_analyse<1, DETAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s1)));
    DS_CUDA(cudaFuncSetAttribute(k1_analyse<4, DETAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(s4)));
    int occ1 = 0, occ4 = 0;
    DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k1_analyse<1, DETAIL>, 32 * kWarpsSmall, s1));
    DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4, k1_analyse<4, DETAIL>, 32 * kWarpsBig, s4));
    if (occ1 < 1 || occ4 < 1) return fail(DS_ECUDA, "analysis kernel does not fit on an SM");
    cfg.grid_small = sms * occ1;  // persistent: one full wave, warps stride over DAGs
    cfg.grid_big = sms * occ4;
    if (slot < 64) {
        cache[slot] = cfg;
        ready[slot] = true;
    }
    return DS_OK;
}

template <bool DETAIL>
int launch_k1(const K1Args& a, const LaunchCfg& cfg, bool any_big, cudaStream_t s) {
    if (a.n_dags == 0) return DS_OK;
    const u64 need_small = (a.n_dags + kWarpsSmall - 1) / kWarpsSmall;
    const int gs = int(std::min<u64>(cfg.grid_small, need_small));
    k1_analyse<1, DETAIL><<<gs, 32 * kWarpsSmall, smem_bytes<1, DETAIL>(kWarpsSmall), s>>>(a);
    DS_CUDA(cudaGetLastError());
    if (any_big) {
        const int gb = int(std::min<u64>(cfg.grid_big, a.n_dags));
        k1_analyse<4, DETAIL><<<gb, 32 * kWarpsBig, smem_bytes<4, DETAIL>(kWarpsBig), s>>>(a);
        DS_CUDA(cudaGetLastError());
    }
    return DS_OK;
}

bool batch_has_big(const uint32_t* node_off, u64 lo, u64 hi) {
    for (u64 d = lo; d < hi; ++d) {
        if (node_off[d + 1] - node_off[d] > 64) return true;
    }
    return false;
}

// ------------------------------------------------------ chunked host path
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap) return DS_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (bytes == 0) return DS_OK;
        DS_CUDA(cudaMalloc(&p, bytes));
        cap = bytes;
        return DS_OK;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct Slot {
    cudaStream_t s = nullptr;
    DevBuf node_off, edge_off, ln, ldn, edges, status, bounds, ngroups;
};

struct DeviceCtx {
    std::mutex mu;
    bool init = false;
    Slot slot[3];
};

DeviceCtx& device_ctx(int dev) {
    static DeviceCtx ctx[64];
    return ctx[dev & 63];
}

int analyze_host(const ds_dag_batch* b, const Plat& P, uint32_t mask, ds_results* out, int device) {
    DS_CUDA(cudaSetDevice(device));
    LaunchCfg cfg;
    if (int rc = configure<false>(device, cfg)) return rc;
    DeviceCtx& ctx = device_ctx(device);
    std::lock_guard<std::mutex> lock(ctx.mu);
    if (!ctx.init) {
        for (auto& sl : ctx.slot) DS_CUDA(cudaStreamCreateWithFlags(&sl.s, cudaStreamNonBlocking));
        ctx.init = true;
    }
    // chunks of ~64k DAGs (>= one wave of warps, small enough to pipeline)
    const u64 chunk = 1ull << 16;
    const u64 n = b->n_dags;
    for (u64 lo = 0, c = 0; lo < n; lo += chunk, ++c) {
        const u64 hi = std::min(n, lo + chunk), nd = hi - lo;
        Slot& sl = ctx.slot[c % 3];
        // indices are relative to node_off[0] / edge_off[0] (header contract)
        const u32 n0 = b->node_off[lo] - b->node_off[0], n1 = b->node_off[hi] - b->node_off[0];
        const u32 e0 = b->edge_off[lo] - b->edge_off[0], e1 = b->edge_off[hi] - b->edge_off[0];
        const size_t nn = n1 - n0, ne = e1 - e0;
        // a slot's buffers are reused: wait for its previous chunk
        DS_CUDA(cudaStreamSynchronize(sl.s));
        if (int rc = sl.node_off.ensure((nd + 1) * 4)) return rc;
        if (int rc = sl.edge_off.ensure((nd + 1) * 4)) return rc;
        if (int rc = sl.ln.ensure(std::max<size_t>(nn, 1) * 8)) return rc;
        if (b->load_den) {
            if (int rc = sl.ldn.ensure(std::max<size_t>(nn, 1) * 8)) return rc;
        }
        if (int rc = sl.edges.ensure(std::max<size_t>(ne, 1) * 4)) return rc;
        if (int rc = sl.status.ensure(nd * 4)) return rc;
        if (int rc = sl.bounds.ensure(nd * 80)) return rc;
        if (int rc = sl.ngroups.ensure(nd * 2)) return rc;
        DS_CUDA(cudaMemcpyAsync(sl.node_off.p, b->node_off + lo, (nd + 1) * 4, cudaMemcpyHostToDevice, sl.s));
        DS_CUDA(cudaMemcpyAsync(sl.edge_off.p, b->edge_off + lo, (nd + 1) * 4, cudaMemcpyHostToDevice, sl.s));
        DS_CUDA(cudaMemcpyAsync(sl.ln.p, b->load_num + n0, nn * 8, cudaMemcpyHostToDevice, sl.s));
        if (b->load_den) {
            DS_CUDA(cudaMemcpyAsync(sl.ldn.p, b->load_den + n0, nn * 8, cudaMemcpyHostToDevice, sl.s));
        }
        DS_CUDA(cudaMemcpyAsync(sl.edges.p, b->edges + e0, ne * 4, cudaMemcpyHostToDevice, sl.s));
        K1Args a{};
        a.n_dags = nd;
        a.node_off = static_cast<const u32*>(sl.node_off.p);
        a.edge_off = static_cast<const u32*>(sl.edge_off.p);
        a.load_num = static_cast<const u64*>(sl.ln.p);
        a.load_den = b->load_den ? static_cast<const u64*>(sl.ldn.p) : nullptr;
        a.edges = static_cast<const u32*>(sl.edges.p);
        a.plat = P;
        a.mask = mask;
        a.status = static_cast<int32_t*>(sl.status.p);
        a.bounds = static_cast<int64_t*>(sl.bounds.p);
        a.n_groups = out->n_groups ? static_cast<uint16_t*>(sl.ngroups.p) : nullptr;
        if (int rc = launch_k1<false>(a, cfg, batch_has_big(b->node_off, lo, hi), sl.s)) return rc;
        DS_CUDA(cudaMemcpyAsync(out->status + lo, sl.status.p, nd * 4, cudaMemcpyDeviceToHost, sl.s));
        DS_CUDA(cudaMemcpyAsync(out->bounds + 10 * lo, sl.bounds.p, nd * 80, cudaMemcpyDeviceToHost, sl.s));
        if (out->n_groups) {
            DS_CUDA(cudaMemcpyAsync(out->n_groups + lo, sl.ngroups.p, nd * 2, cudaMemcpyDeviceToHost, sl.s));
        }
    }
    for (auto& sl : ctx.slot) DS_CUDA(cudaStreamSynchronize(sl.s));
    return DS_OK;
}

// ------------------------------------------------------------------ session
struct Session {
    int device = 0;
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    DevBuf node_off, edge_off, ln, ldn, edges, status, bounds, ngroups;
    K1Args args{};
    LaunchCfg cfg;
    bool any_big = false;
    u64 n_dags = 0;
};

}  // namespace ds

using namespace ds;

extern "C" {

const char* ds_last_error(void) { return g_err.c_str(); }
const char* ds_version(void) { return "dagsched_b200 0.1 (sm_100a)"; }

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

int ds_analyze_batch(const ds_dag_batch* batch, const ds_platform* platform, uint32_t method_mask,
                     ds_results* out, int device, void* stream, uint32_t flags) {
    if (!batch || !out || !out->status || !out->bounds) return fail(DS_EINVAL, "NULL batch or results");
    Plat P;
    if (int rc = check_platform(platform, P)) return rc;
    if (batch->n_dags == 0) return DS_OK;
    if (!(flags & DS_F_DEVICE_PTRS)) return analyze_host(batch, P, method_mask & DS_M_ALL, out, device);
    DS_CUDA(cudaSetDevice(device));
    LaunchCfg cfg;
    if (int rc = configure<false>(device, cfg)) return rc;
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
    // device pointers: size classes unknown on the host, so the n<=256 kernel
    // always runs (it skips DAGs with n <= 64 after two offset loads)
    return launch_k1<false>(a, cfg, true, static_cast<cudaStream_t>(stream));
}

int ds_analyze_batch_multi(const ds_dag_batch* batch, const ds_platform* platform, uint32_t method_mask,
                           ds_results* out, const int* devices, int n_devices) {
    if (!batch || !out || !devices || n_devices < 1) return fail(DS_EINVAL, "bad arguments");
    const u64 n = batch->n_dags;
    std::vector<int> rcs(n_devices, DS_OK);
    std::vector<std::string> errs(n_devices);
    std::vector<std::thread> th;
    for (int i = 0; i < n_devices; ++i) {
        const u64 lo = n * u64(i) / u64(n_devices), hi = n * u64(i + 1) / u64(n_devices);
        th.emplace_back([&, i, lo, hi] {
            ds_dag_batch sub = *batch;
            sub.n_dags = hi - lo;
            sub.node_off = batch->node_off + lo;
            sub.edge_off = batch->edge_off + lo;
            sub.load_num = batch->load_num + (batch->node_off[lo] - batch->node_off[0]);
            sub.load_den = batch->load_den ? batch->load_den + (batch->node_off[lo] - batch->node_off[0]) : nullptr;
            sub.edges = batch->edges + (batch->edge_off[lo] - batch->edge_off[0]);
            ds_results r = *out;
            r.status = out->status + lo;
            r.bounds = out->bounds + 10 * lo;
            r.n_groups = out->n_groups ? out->n_groups + lo : nullptr;
            rcs[i] = ds_analyze_batch(&sub, platform, method_mask, &r, devices[i], nullptr, 0);
            errs[i] = g_err;
        });
    }
    for (auto& t : th) t.join();
    for (int i = 0; i < n_devices; ++i) {
        if (rcs[i] != DS_OK) return fail(rcs[i], errs[i]);
    }
    return DS_OK;
}

int ds_schedule_batch(const ds_dag_batch* b, const ds_platform* platform, ds_scheme_out* out, int device) {
    if (!b || !out) return fail(DS_EINVAL, "NULL batch or output");
    Plat P;
    if (int rc = check_platform(platform, P)) return rc;
    const u64 n = b->n_dags;
    if (n == 0) return DS_OK;
    DS_CUDA(cudaSetDevice(device));
    LaunchCfg cfg;
    if (int rc = configure<true>(device, cfg)) return rc;
    const u32 n0 = b->node_off[0], N = b->node_off[n] - n0;
    const u32 e0 = b->edge_off[0], E = b->edge_off[n] - e0;
    DevBuf node_off, edge_off, ln, ldn, edges, status, ne, ng, nd, nb, ndg, ent, grp, bounds;
    if (int rc = node_off.ensure((n + 1) * 4)) return rc;
    if (int rc = edge_off.ensure((n + 1) * 4)) return rc;
    if (int rc = ln.ensure(std::max<u32>(N, 1) * 8)) return rc;
    if (int rc = ldn.ensure(std::max<u32>(N, 1) * 8)) return rc;
    if (int rc = edges.ensure(std::max<u32>(E, 1) * 4)) return rc;
    if (int rc = status.ensure(n * 4)) return rc;
    if (int rc = ne.ensure(n * 2)) return rc;
    if (int rc = ng.ensure(n * 2)) return rc;
    if (int rc = nd.ensure(n * 2)) return rc;
    if (int rc = nb.ensure(std::max<u32>(N, 1) * 2)) return rc;
    if (int rc = ndg.ensure(std::max<u32>(N, 1) * 2)) return rc;
    if (int rc = ent.ensure(std::max<u32>(2 * N, 1) * sizeof(ds_entity_rec))) return rc;
    if (int rc = grp.ensure(std::max<u32>(N, 1) * sizeof(ds_group_rec))) return rc;
    if (int rc = bounds.ensure(n * 80)) return rc;
    std::vector<u32> no(n + 1), eo(n + 1);
    for (u64 i = 0; i <= n; ++i) {
        no[i] = b->node_off[i] - n0;
        eo[i] = b->edge_off[i] - e0;
    }
    DS_CUDA(cudaMemcpy(node_off.p, no.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
    DS_CUDA(cudaMemcpy(edge_off.p, eo.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
    DS_CUDA(cudaMemcpy(ln.p, b->load_num, size_t(N) * 8, cudaMemcpyHostToDevice));
    if (b->load_den) DS_CUDA(cudaMemcpy(ldn.p, b->load_den, size_t(N) * 8, cudaMemcpyHostToDevice));
    DS_CUDA(cudaMemcpy(edges.p, b->edges, size_t(E) * 4, cudaMemcpyHostToDevice));
    DS_CUDA(cudaMemset(nb.p, 0xff, std::max<u32>(N, 1) * 2));
    DS_CUDA(cudaMemset(ndg.p, 0xff, std::max<u32>(N, 1) * 2));
    DS_CUDA(cudaMemset(ent.p, 0, std::max<u32>(2 * N, 1) * sizeof(ds_entity_rec)));
    DS_CUDA(cudaMemset(grp.p, 0, std::max<u32>(N, 1) * sizeof(ds_group_rec)));
    K1Args a{};
    a.n_dags = n;
    a.node_off = static_cast<const u32*>(node_off.p);
    a.edge_off = static_cast<const u32*>(edge_off.p);
    a.load_num = static_cast<const u64*>(ln.p);
    a.load_den = b->load_den ? static_cast<const u64*>(ldn.p) : nullptr;
    a.edges = static_cast<const u32*>(edges.p);
    a.plat = P;
    a.mask = DS_M_ALL;
    a.det.status = static_cast<int32_t*>(status.p);
    a.det.n_entities = static_cast<uint16_t*>(ne.p);
    a.det.n_groups = static_cast<uint16_t*>(ng.p);
    a.det.n_div_groups = static_cast<uint16_t*>(nd.p);
    a.det.node_block = static_cast<int16_t*>(nb.p);
    a.det.node_div_group = static_cast<int16_t*>(ndg.p);
    a.det.entities = static_cast<ds_entity_rec*>(ent.p);
    a.det.groups = static_cast<ds_group_rec*>(grp.p);
    a.det.bounds = static_cast<int64_t*>(bounds.p);
    if (int rc = launch_k1<true>(a, cfg, batch_has_big(b->node_off, 0, n), nullptr)) return rc;
    DS_CUDA(cudaDeviceSynchronize());
    if (out->status) DS_CUDA(cudaMemcpy(out->status, status.p, n * 4, cudaMemcpyDeviceToHost));
    if (out->n_entities) DS_CUDA(cudaMemcpy(out->n_entities, ne.p, n * 2, cudaMemcpyDeviceToHost));
    if (out->n_groups) DS_CUDA(cudaMemcpy(out->n_groups, ng.p, n * 2, cudaMemcpyDeviceToHost));
    if (out->n_div_groups) DS_CUDA(cudaMemcpy(out->n_div_groups, nd.p, n * 2, cudaMemcpyDeviceToHost));
    if (out->node_block) DS_CUDA(cudaMemcpy(out->node_block, nb.p, size_t(N) * 2, cudaMemcpyDeviceToHost));
    if (out->node_div_group)
        DS_CUDA(cudaMemcpy(out->node_div_group, ndg.p, size_t(N) * 2, cudaMemcpyDeviceToHost));
    if (out->entities)
        DS_CUDA(cudaMemcpy(out->entities, ent.p, size_t(2) * N * sizeof(ds_entity_rec), cudaMemcpyDeviceToHost));
    if (out->groups)
        DS_CUDA(cudaMemcpy(out->groups, grp.p, size_t(N) * sizeof(ds_group_rec), cudaMemcpyDeviceToHost));
    if (out->bounds) DS_CUDA(cudaMemcpy(out->bounds, bounds.p, n * 80, cudaMemcpyDeviceToHost));
    return DS_OK;
}

int ds_session_create(const ds_dag_batch* b, const ds_platform* platform, uint32_t method_mask, int device,
                      void** session) {
    if (!b || !session) return fail(DS_EINVAL, "NULL argument");
    Plat P;
    if (int rc = check_platform(platform, P)) return rc;
    auto* S = new Session();
    S->device = device;
    S->n_dags = b->n_dags;
    auto bail = [&](int rc) {
        delete S;
        return rc;
    };
    if (cudaSetDevice(device) != cudaSuccess) return bail(fail(DS_ECUDA, "cudaSetDevice"));
    if (int rc = configure<false>(device, S->cfg)) return bail(rc);
    const u64 n = b->n_dags;
    const u32 n0 = b->node_off[0], N = b->node_off[n] - n0;
    const u32 e0 = b->edge_off[0], E = b->edge_off[n] - e0;
    std::vector<u32> no(n + 1), eo(n + 1);
    for (u64 i = 0; i <= n; ++i) {
        no[i] = b->node_off[i] - n0;
        eo[i] = b->edge_off[i] - e0;
    }
    S->any_big = batch_has_big(b->node_off, 0, n);
    int rc = DS_OK;
    rc = rc ? rc : S->node_off.ensure((n + 1) * 4);
    rc = rc ? rc : S->edge_off.ensure((n + 1) * 4);
    rc = rc ? rc : S->ln.ensure(std::max<u32>(N, 1) * 8);
    rc = rc ? rc : (b->load_den ? S->ldn.ensure(std::max<u32>(N, 1) * 8) : DS_OK);
    rc = rc ? rc : S->edges.ensure(std::max<u32>(E, 1) * 4);
    rc = rc ? rc : S->status.ensure(std::max<u64>(n, 1) * 4);
    rc = rc ? rc : S->bounds.ensure(std::max<u64>(n, 1) * 80);
    rc = rc ? rc : S->ngroups.ensure(std::max<u64>(n, 1) * 2);
    if (rc) return bail(rc);
    if (cudaStreamCreateWithFlags(&S->s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&S->e0) != cudaSuccess || cudaEventCreate(&S->e1) != cudaSuccess ||
        cudaMemcpy(S->node_off.p, no.data(), (n + 1) * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(S->edge_off.p, eo.data(), (n + 1) * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(S->ln.p, b->load_num, size_t(N) * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
        (b->load_den &&
         cudaMemcpy(S->ldn.p, b->load_den, size_t(N) * 8, cudaMemcpyHostToDevice) != cudaSuccess) ||
        cudaMemcpy(S->edges.p, b->edges, size_t(E) * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
        return bail(fail(DS_ECUDA, std::string("session upload: ") + cudaGetErrorString(cudaGetLastError())));
    }
    K1Args& a = S->args;
    a.n_dags = n;
    a.node_off = static_cast<const u32*>(S->node_off.p);
    a.edge_off = static_cast<const u32*>(S->edge_off.p);
    a.load_num = static_cast<const u64*>(S->ln.p);
    a.load_den = b->load_den ? static_cast<const u64*>(S->ldn.p) : nullptr;
    a.edges = static_cast<const u32*>(S->edges.p);
    a.plat = P;
    a.mask = method_mask & DS_M_ALL;
    a.status = static_cast<int32_t*>(S->status.p);
    a.bounds = static_cast<int64_t*>(S->bounds.p);
    a.n_groups = static_cast<uint16_t*>(S->ngroups.p);
    *session = S;
    return DS_OK;
}

int ds_session_run(void* session, float* kernel_ms) {
    auto* S = static_cast<Session*>(session);
    DS_CUDA(cudaSetDevice(S->device));
    DS_CUDA(cudaEventRecord(S->e0, S->s));
    if (int rc = launch_k1<false>(S->args, S->cfg, S->any_big, S->s)) return rc;
    DS_CUDA(cudaEventRecord(S->e1, S->s));
    DS_CUDA(cudaEventSynchronize(S->e1));
    if (kernel_ms) DS_CUDA(cudaEventElapsedTime(kernel_ms, S->e0, S->e1));
    return DS_OK;
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
    if (S->e0) cudaEventDestroy(S->e0);
    if (S->e1) cudaEventDestroy(S->e1);
    if (S->s) cudaStreamDestroy(S->s);
    delete S;
    return DS_OK;
}

}  // extern "C"

// K6 launcher + C-ABI entry (ds_simulate_greedy_batch).
#include <algorithm>
#include <string>
#include <vector>

#include "k6_greedy.cuh"

namespace ds {
int fail(int code, const std::string& msg);
}

using namespace ds;

#define K6_CUDA(call)                                                                                   \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) return fail(DS_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

namespace {
struct Buf {
    void* p = nullptr;
    ~Buf() {
        if (p) cudaFree(p);
    }
};
// FactorSource (simulator.cpp:18-34): lo = max(1, ceil(smin*1024)), hi = max(lo, floor(smax*1024))
bool factor_bounds(const ds_greedy_cfg* c, long long& lo, long long& hi) {
    lo = hi = 1024;
    if (!c->scaled) return true;
    if (c->scale_min_den <= 0 || c->scale_max_den <= 0) return false;
    const __int128 a = c->scale_min_num, b = c->scale_min_den, x = c->scale_max_num, y = c->scale_max_den;
    if (a <= 0 || x > y || a * y > x * b) return false;  // 0 < min <= max <= 1
    const __int128 n1 = a * 1024, n2 = x * 1024;
    lo = (long long)((n1 + b - 1) / b);
    hi = (long long)(n2 / y);
    if (lo < 1) lo = 1;
    if (hi < lo) hi = lo;
    return true;
}
}  // namespace

extern "C" int ds_simulate_greedy_batch(const ds_dag_batch* b, const ds_platform* plat, const ds_greedy_cfg* cfg,
                                        int32_t* status, int64_t* makespan, int64_t* events, int device) {
    if (!b || !plat || !cfg || !status || !makespan) return fail(DS_EINVAL, "NULL argument");
    if (plat->sm_count <= 0) return fail(DS_EINVAL, "sm_count must be positive");
    if (plat->tmin_num <= 0 || plat->tmin_den <= 0) return fail(DS_EINVAL, "t_min must be positive");
    if (cfg->runs < 1) return fail(DS_EINVAL, "runs must be >= 1");
    if (cfg->policy != 0 && cfg->policy != 1) return fail(DS_EINVAL, "policy must be fifo (0) or random (1)");
    K6Args a{};
    if (!factor_bounds(cfg, a.lo, a.hi)) return fail(DS_EINVAL, "scale factors must satisfy 0 < min <= max <= 1");
    const u64 n = b->n_dags;
    if (n == 0) return DS_OK;
    const u64 nb = b->node_off[0], eb = b->edge_off[0];
    const u64 N = b->node_off[n] - nb, E = b->edge_off[n] - eb;
    const u64 P = n * u64(cfg->runs);
    bool big = false, huge = false;
    std::vector<u32> no(n + 1), eo(n + 1);
    for (u64 i = 0; i <= n; ++i) {
        no[i] = u32(b->node_off[i] - nb);
        eo[i] = u32(b->edge_off[i] - eb);
        if (i && no[i] - no[i - 1] > 64) big = true;
        if (i && no[i] - no[i - 1] > 256) huge = true;
    }
    K6_CUDA(cudaSetDevice(device));
    cudaStream_t s;
    K6_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    Buf dno, deo, dln, dld, ded, dst, dmk, dev, dscr;
    K6_CUDA(cudaMalloc(&dno.p, (n + 1) * 4));
    K6_CUDA(cudaMalloc(&deo.p, (n + 1) * 4));
    K6_CUDA(cudaMalloc(&dln.p, std::max<u64>(N, 1) * 8));
    if (b->load_den) K6_CUDA(cudaMalloc(&dld.p, std::max<u64>(N, 1) * 8));
    K6_CUDA(cudaMalloc(&ded.p, std::max<u64>(E, 1) * 4));
    K6_CUDA(cudaMalloc(&dst.p, P * 4));
    K6_CUDA(cudaMalloc(&dmk.p, P * 16));
    if (events) K6_CUDA(cudaMalloc(&dev.p, std::max<u64>(N, 1) * cfg->runs * 32));
    K6_CUDA(cudaMemcpyAsync(dno.p, no.data(), (n + 1) * 4, cudaMemcpyHostToDevice, s));
    K6_CUDA(cudaMemcpyAsync(deo.p, eo.data(), (n + 1) * 4, cudaMemcpyHostToDevice, s));
    if (N) K6_CUDA(cudaMemcpyAsync(dln.p, b->load_num, N * 8, cudaMemcpyHostToDevice, s));
    if (N && b->load_den) K6_CUDA(cudaMemcpyAsync(dld.p, b->load_den, N * 8, cudaMemcpyHostToDevice, s));
    if (E) K6_CUDA(cudaMemcpyAsync(ded.p, b->edges, E * 4, cudaMemcpyHostToDevice, s));
    if (events) K6_CUDA(cudaMemsetAsync(dev.p, 0, std::max<u64>(N, 1) * cfg->runs * 32, s));
    a.n_dags = n;
    a.runs = cfg->runs;
    a.node_off = static_cast<const u32*>(dno.p);
    a.edge_off = static_cast<const u32*>(deo.p);
    a.load_num = static_cast<const u64*>(dln.p);
    a.load_den = b->load_den ? static_cast<const u64*>(dld.p) : nullptr;
    a.edges = static_cast<const u32*>(ded.p);
    a.M = plat->sm_count;
    a.tmin_n = u64(plat->tmin_num);
    a.tmin_d = u64(plat->tmin_den);
    a.policy = cfg->policy;
    a.policy_seed = cfg->policy_seed;
    a.scaled = cfg->scaled;
    a.time_seed = cfg->time_seed;
    a.status = static_cast<int32_t*>(dst.p);
    a.makespan = static_cast<int64_t*>(dmk.p);
    a.events = events ? static_cast<int64_t*>(dev.p) : nullptr;
    int sms = 0;
    K6_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    auto grid = [&](u64 cap_per_sm) {
        const u64 need = (P + 63) / 64, cap = u64(sms) * cap_per_sm;
        return unsigned(need < cap ? need : cap);
    };
    k6_greedy<64, u64><<<grid(32), 64, 0, s>>>(a);
    K6_CUDA(cudaGetLastError());
    if (big) {
        k6_greedy<256, u64><<<grid(4), 64, 0, s>>>(a);
        K6_CUDA(cudaGetLastError());
    }
    k6_greedy<256, u128><<<grid(4), 64, 0, s>>>(a);  // the runs that overflowed 64 bits
    K6_CUDA(cudaGetLastError());
    if (huge) {  // n > 256: run state in HBM, one slot per resident thread (u128-sized, ~238 KB)
        K6_CUDA(cudaMalloc(&dscr.p, size_t(kK6BigThreads) * K6Slot<1024, u128>::kBytes));
        a.scratch = static_cast<unsigned char*>(dscr.p);
        const unsigned gb = unsigned(std::min<u64>((P + 31) / 32, kK6BigThreads / 32));
        k6_greedy<1024, u64><<<gb, 32, 0, s>>>(a);
        K6_CUDA(cudaGetLastError());
        k6_greedy<1024, u128><<<gb, 32, 0, s>>>(a);
        K6_CUDA(cudaGetLastError());
    }
    K6_CUDA(cudaMemcpyAsync(status, dst.p, P * 4, cudaMemcpyDeviceToHost, s));
    K6_CUDA(cudaMemcpyAsync(makespan, dmk.p, P * 16, cudaMemcpyDeviceToHost, s));
    if (events) K6_CUDA(cudaMemcpyAsync(events, dev.p, N * cfg->runs * 32, cudaMemcpyDeviceToHost, s));
    K6_CUDA(cudaStreamSynchronize(s));
    return DS_OK;
}

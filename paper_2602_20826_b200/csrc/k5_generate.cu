// K5 launcher: generate_corpus on the device (two replayed passes around a
// 64-bit exclusive scan), then one copy of the packed batch into the
// caller's host arrays (pinned ones make it a single DMA per array).
#include <cub/device/device_scan.cuh>

#include <string>

#include "k5_generate.cuh"
#include "k5_generate_host.h"

namespace ds {

int fail(int code, const std::string& msg);

namespace {
struct AddU64 {
    __device__ __forceinline__ u64 operator()(u64 a, u64 b) const { return a + b; }
};

struct Bufs {  // device scratch, released on every exit path
    void* p[10] = {};
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ~Bufs() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        for (void* q : p)
            if (q) cudaFree(q);
        if (s) cudaStreamDestroy(s);
    }
};
}  // namespace

#define K5_CUDA(call)                                                                                   \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) return fail(DS_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

int k5_generate_host(const K5Params& p, int words, int device, K5Alloc alloc, void* user, float* kernel_ms) {
    K5Args a{};
    a.count = p.count;
    a.seed = p.seed;
    a.dmin = p.dmin;
    a.dmax = p.dmax;
    a.width = p.width;
    a.integer_loads = p.integer_loads;
    a.exact_mean = p.exact_mean;
    a.lo = p.lo;
    a.hi = p.hi;
    a.tmin_f = p.tmin_f;
    a.density = p.density;
    a.tmin_n = p.tmin_n;
    a.tmin_d = p.tmin_d;
    a.avg_n = p.avg_n;
    a.avg_d = p.avg_d;
    const u64 n = a.count;
    K5_CUDA(cudaSetDevice(device));
    Bufs b;
    K5_CUDA(cudaStreamCreateWithFlags(&b.s, cudaStreamNonBlocking));
    K5_CUDA(cudaMalloc(&b.p[0], (n + 1) * 4));  // n_nodes
    K5_CUDA(cudaMalloc(&b.p[1], (n + 1) * 4));  // n_edges
    K5_CUDA(cudaMalloc(&b.p[2], (n + 1) * 8));  // node_off64
    K5_CUDA(cudaMalloc(&b.p[3], (n + 1) * 8));  // edge_off64
    K5_CUDA(cudaMalloc(&b.p[4], 16));           // bad
    a.n_nodes = static_cast<u32*>(b.p[0]);
    a.n_edges = static_cast<u32*>(b.p[1]);
    a.node_off64 = static_cast<const u64*>(b.p[2]);
    a.edge_off64 = static_cast<const u64*>(b.p[3]);
    a.bad = static_cast<int*>(b.p[4]);
    K5_CUDA(cudaMemsetAsync(b.p[0], 0, (n + 1) * 4, b.s));
    K5_CUDA(cudaMemsetAsync(b.p[1], 0, (n + 1) * 4, b.s));
    K5_CUDA(cudaMemsetAsync(b.p[4], 0, 16, b.s));
    K5_CUDA(cudaEventCreate(&b.e0));
    K5_CUDA(cudaEventCreate(&b.e1));
    cudaEvent_t e0 = b.e0, e1 = b.e1;
    K5_CUDA(cudaEventRecord(e0, b.s));
    const unsigned grid = unsigned((n + 127) / 128);
    if (words == 1) k5_generate<1, false><<<grid, 128, 0, b.s>>>(a);
    else k5_generate<4, false><<<grid, 128, 0, b.s>>>(a);
    K5_CUDA(cudaGetLastError());
    size_t tmp = 0;
    K5_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, tmp, a.n_nodes, static_cast<u64*>(b.p[2]), AddU64(), u64(0),
                                           n + 1, b.s));
    K5_CUDA(cudaMalloc(&b.p[5], tmp));
    K5_CUDA(cub::DeviceScan::ExclusiveScan(b.p[5], tmp, a.n_nodes, static_cast<u64*>(b.p[2]), AddU64(), u64(0),
                                           n + 1, b.s));
    K5_CUDA(cub::DeviceScan::ExclusiveScan(b.p[5], tmp, a.n_edges, static_cast<u64*>(b.p[3]), AddU64(), u64(0),
                                           n + 1, b.s));
    u64 tot[2];
    K5_CUDA(cudaMemcpyAsync(&tot[0], a.node_off64 + n, 8, cudaMemcpyDeviceToHost, b.s));
    K5_CUDA(cudaMemcpyAsync(&tot[1], a.edge_off64 + n, 8, cudaMemcpyDeviceToHost, b.s));
    K5_CUDA(cudaStreamSynchronize(b.s));
    if (tot[0] > 0xffffffffull || tot[1] > 0xffffffffull)
        return fail(DS_ETOOBIG, "batch exceeds 2^32 nodes or edges");
    K5_CUDA(cudaMalloc(&b.p[6], (n + 1) * 4));                // node_off
    K5_CUDA(cudaMalloc(&b.p[7], (n + 1) * 4));                // edge_off
    K5_CUDA(cudaMalloc(&b.p[8], std::max<u64>(tot[1], 1) * 4));  // edges
    K5_CUDA(cudaMalloc(&b.p[9], std::max<u64>(tot[0], 1) * 16)); // loads (num | den)
    a.node_off = static_cast<u32*>(b.p[6]);
    a.edge_off = static_cast<u32*>(b.p[7]);
    a.edges = static_cast<u32*>(b.p[8]);
    a.load_num = static_cast<int64_t*>(b.p[9]);
    a.load_den = a.load_num + tot[0];
    if (words == 1) k5_generate<1, true><<<grid, 128, 0, b.s>>>(a);
    else k5_generate<4, true><<<grid, 128, 0, b.s>>>(a);
    K5_CUDA(cudaGetLastError());
    K5_CUDA(cudaEventRecord(e1, b.s));
    K5Host h{};
    const int rc = alloc(tot[0], tot[1], user, &h);
    if (rc != DS_OK) return rc;
    int bad = 0;
    K5_CUDA(cudaMemcpyAsync(h.node_off, a.node_off, (n + 1) * 4, cudaMemcpyDeviceToHost, b.s));
    K5_CUDA(cudaMemcpyAsync(h.edge_off, a.edge_off, (n + 1) * 4, cudaMemcpyDeviceToHost, b.s));
    if (tot[1]) K5_CUDA(cudaMemcpyAsync(h.edges, a.edges, tot[1] * 4, cudaMemcpyDeviceToHost, b.s));
    if (tot[0]) {
        K5_CUDA(cudaMemcpyAsync(h.load_num, a.load_num, tot[0] * 8, cudaMemcpyDeviceToHost, b.s));
        K5_CUDA(cudaMemcpyAsync(h.load_den, a.load_den, tot[0] * 8, cudaMemcpyDeviceToHost, b.s));
    }
    K5_CUDA(cudaMemcpyAsync(&bad, a.bad, 4, cudaMemcpyDeviceToHost, b.s));
    K5_CUDA(cudaStreamSynchronize(b.s));
    if (kernel_ms) K5_CUDA(cudaEventElapsedTime(kernel_ms, e0, e1));
    if (bad) return fail(DS_EOVERFLOW, "generated load outside int64");
    return DS_OK;
}

}  // namespace ds

// Platform-stall probe: does the GPU stop running this context for ~ms at a
// time? One CTA per requested SM spins reading %globaltimer for `secs`
// seconds and records every gap between consecutive reads above
// `thresh_us`; a gap seen by every SM at once means the whole context was
// off the GPU (time-slicing with another context, or a driver pause), not a
// slow kernel. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o
// tools/heartbeat tools/heartbeat.cu ; run: tools/heartbeat [secs] [ctas]
// [thresh_us]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}

constexpr int kMaxGaps = 4096;

__global__ void spin(unsigned long long dur_ns, unsigned long long thresh_ns, unsigned long long* gaps,
                     unsigned* n_gaps, unsigned* sm) {
    if (threadIdx.x) return;
    const unsigned long long t0 = gtime();
    unsigned long long prev = t0;
    sm[blockIdx.x] = smid();
    for (;;) {
        const unsigned long long t = gtime();
        if (t - prev > thresh_ns) {
            const unsigned i = atomicAdd(n_gaps, 1u);
            if (i < kMaxGaps) {
                gaps[3 * i] = prev - t0;
                gaps[3 * i + 1] = t - prev;
                gaps[3 * i + 2] = blockIdx.x;
            }
        }
        prev = t;
        if (t - t0 > dur_ns) break;
    }
}

int main(int argc, char** argv) {
    const double secs = argc > 1 ? atof(argv[1]) : 5.0;
    const int ctas = argc > 2 ? atoi(argv[2]) : 4;
    const double thresh_us = argc > 3 ? atof(argv[3]) : 50.0;
    unsigned long long* gaps;
    unsigned *n, *sm;
    cudaMalloc(&gaps, kMaxGaps * 3 * 8);
    cudaMalloc(&n, 4);
    cudaMalloc(&sm, ctas * 4);
    cudaMemset(n, 0, 4);
    spin<<<ctas, 32>>>((unsigned long long)(secs * 1e9), (unsigned long long)(thresh_us * 1e3), gaps, n, sm);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
        return 1;
    }
    unsigned hn = 0;
    cudaMemcpy(&hn, n, 4, cudaMemcpyDeviceToHost);
    std::vector<unsigned long long> g(kMaxGaps * 3);
    std::vector<unsigned> s(ctas);
    cudaMemcpy(g.data(), gaps, g.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(s.data(), sm, ctas * 4, cudaMemcpyDeviceToHost);
    printf("{\"secs\": %.1f, \"ctas\": %d, \"thresh_us\": %.0f, \"n_gaps\": %u, \"sms\": [", secs, ctas, thresh_us, hn);
    for (int i = 0; i < ctas; ++i) printf("%s%u", i ? ", " : "", s[i]);
    printf("], \"gaps\": [");
    for (unsigned i = 0; i < hn && i < kMaxGaps; ++i)
        printf("%s[%.3f, %.1f, %llu]", i ? ", " : "", g[3 * i] / 1e6, g[3 * i + 1] / 1e3, g[3 * i + 2]);
    printf("]}\n");
    return 0;
}

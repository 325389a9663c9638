// Host-side interface of K5 (device corpus generation), shared by the g++
// translation unit (host_gen.cpp) and the nvcc one (k5_generate.cu).
#pragma once

#include <stdint.h>

namespace ds {

struct K5Params {  // GenConfig, pre-digested on the host like generator.cpp:24-96
    uint64_t count, seed;
    int dmin, dmax, width, integer_loads, exact_mean;
    double lo, hi, tmin_f, density;
    uint64_t tmin_n, tmin_d, avg_n, avg_d;  // reduced
};

struct K5Host {  // the caller's host arrays for the packed batch
    uint32_t *node_off, *edge_off, *edges;
    int64_t *load_num, *load_den;
};
// Called once the totals are known; fills *out (DS_OK) or returns an error.
typedef int (*K5Alloc)(uint64_t nn, uint64_t ne, void* user, K5Host* out);

// Generates p.count DAGs on `device` (successor masks of `words` x 64 bits)
// and copies the packed batch into the arrays alloc provides.
int k5_generate_host(const K5Params& p, int words, int device, K5Alloc alloc, void* user, float* kernel_ms);

}  // namespace ds

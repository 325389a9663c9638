// libstdc++'s std::mt19937_64 and uniform_int_distribution on the device,
// shared by K4 (validation) and K5 (generation).
#pragma once

#include "rat.cuh"

namespace ds {

struct Mt64 {
    static constexpr int N = 312, M = 156;
    u64 mt[N];
    int i;
    __device__ void seed(u64 s) {
        mt[0] = s;
        for (int k = 1; k < N; ++k) mt[k] = 6364136223846793005ull * (mt[k - 1] ^ (mt[k - 1] >> 62)) + u64(k);
        i = N;
    }
    __device__ void twist() {
        constexpr u64 upper = ~((1ull << 31) - 1), lower = (1ull << 31) - 1, a = 0xB5026F5AA96619E9ull;
        for (int k = 0; k < N; ++k) {
            const u64 x = (mt[k] & upper) | (mt[(k + 1) % N] & lower);
            mt[k] = mt[(k + M) % N] ^ (x >> 1) ^ ((x & 1ull) ? a : 0ull);
        }
        i = 0;
    }
    __device__ u64 next() {
        if (i >= N) twist();
        u64 y = mt[i++];
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        y ^= y >> 43;
        return y;
    }
};

// uniform_int_distribution<long long>(lo, hi)(mt19937_64) as libstdc++ 13.
__device__ __forceinline__ long long uniform_ll(Mt64& g, long long lo, long long hi) {
    const u64 range = u64(hi) - u64(lo) + 1;  // __uerange; hi > lo - 1 always here
    u128 prod = u128(g.next()) * range;
    u64 low = u64(prod);
    if (low < range) {
        const u64 threshold = (0ull - range) % range;
        while (low < threshold) {
            prod = u128(g.next()) * range;
            low = u64(prod);
        }
    }
    return (long long)(u64(prod >> 64)) + lo;
}

}  // namespace ds

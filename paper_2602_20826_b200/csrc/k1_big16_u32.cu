// k1_big, W = 16 (512 < n <= 1024), u32 words, bounds and detail mode (one TU
// per word type: each W = 16 instantiation takes ~80 s of ptxas).
#include "k1_big.cuh"

namespace ds {
DS_K1_BIG_INSTANCE(16, u32, false, k1_big_16_u32_b)
DS_K1_BIG_INSTANCE(16, u32, true, k1_big_16_u32_d)
}  // namespace ds

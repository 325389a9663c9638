// k1_big, W = 8 (256 < n <= 512): all word tiers, bounds and detail mode.
#include "k1_big.cuh"

namespace ds {
DS_K1_BIG_INSTANCE(8, u32, false, k1_big_8_u32_b)
DS_K1_BIG_INSTANCE(8, u64, false, k1_big_8_u64_b)
DS_K1_BIG_INSTANCE(8, u128, false, k1_big_8_u128_b)
DS_K1_BIG_INSTANCE(8, u32, true, k1_big_8_u32_d)
DS_K1_BIG_INSTANCE(8, u64, true, k1_big_8_u64_d)
DS_K1_BIG_INSTANCE(8, u128, true, k1_big_8_u128_d)
}  // namespace ds

// K4 instantiation + launcher (batched run_validation).
#include "k4_validate.cuh"

namespace ds {

void k4_launch(u64 n_dags, const u32* node_off, const int32_t* status, const uint16_t* n_groups,
               const ds_group_rec* groups, const ds_entity_rec* ents, const int64_t* bounds, int samples,
               long long lo, long long hi, u64 seed, unsigned char* over, double* ratio, int32_t* st,
               cudaStream_t stream) {
    K4Args a{n_dags, node_off, status, n_groups, groups, ents, bounds, samples, lo, hi, seed, over, ratio, st};
    const u64 T = n_dags * (u64(samples) + 1);
    k4_validate<<<unsigned((T + 127) / 128), 128, 0, stream>>>(a);
}

}  // namespace ds

// K4 — batched Theorem-1 validation: the device twin of run_validation
// (experiment.cpp:163-240) over simulate_scheme (simulator.cpp:14-94).
//
// One thread per (DAG, sample). Sample s < S replays the DAG's schedule with
// every entity's duration scaled by a factor k/1024 drawn from
// uniform_int_distribution<long long>(lo, hi) over std::mt19937_64 seeded with
// seed + 7919 * d + s — libstdc++'s exact algorithms (mt19937_64 twist and
// tempering; Lemire's nearly-divisionless downscaling with a 128-bit product,
// /usr/include/c++/13/bits/uniform_int_dist.h:252-328), in simulate_scheme's
// draw order (per group: members, then launches). Sample s == S is the worst
// case (factor 1). Group windows close when their longest entity ends; the
// makespan is their exact sum, compared exactly with the bound; the ratio is
// makespan / bound reduced and converted to double like to_double().
#pragma once

#include "../../include/dagsched_b200.h"
#include "rat.cuh"
#include "rng.cuh"

namespace ds {

struct K4Args {
    u64 n_dags;
    const u32* node_off;       // rebased, for the detail slot bases
    const int32_t* status;     // K1 detail status
    const uint16_t* n_groups;
    const ds_group_rec* groups;
    const ds_entity_rec* ents;
    const int64_t* bounds;     // proposed bound at slot 0
    int samples;               // S scaled samples (+1 worst case per DAG)
    long long lo, hi;          // factor grid bounds (1/1024 units)
    u64 seed;                  // config.seed
    unsigned char* over;       // [n_dags * (S + 1)] makespan > bound
    double* ratio;             // [n_dags * (S + 1)] makespan / bound
    int32_t* st;               // [n_dags * (S + 1)] DS_OK / DS_EOVERFLOW / K1 status
};

__global__ void __launch_bounds__(128) k4_validate(const K4Args a) {
    const u64 per = u64(a.samples) + 1;
    const u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= a.n_dags * per) return;
    const u64 d = t / per;
    const int s = int(t % per);
    if (a.status[d] != DS_OK) {
        a.st[t] = a.status[d];
        a.over[t] = 0;
        a.ratio[t] = 0.0;
        return;
    }
    const bool worst = s == a.samples;
    Mt64 g;
    if (!worst) g.seed(a.seed + 7919ull * d + u64(s));
    const ds_group_rec* G = a.groups + a.node_off[d];
    const ds_entity_rec* E = a.ents + 2ull * a.node_off[d];
    bool ovf = false;
    RatT<u128> clock{0, 1};
    for (int j = 0; j < a.n_groups[d]; ++j) {
        const ds_group_rec& gr = G[j];
        RatT<u128> window{0, 1};
        // simulate_scheme draws members first, then launches
        for (int pass = 0; pass < 2; ++pass) {
            const int b0 = pass == 0 ? gr.first_entity + gr.n_launches : gr.first_entity;
            const int cnt = pass == 0 ? gr.n_members : gr.n_launches;
            for (int k = 0; k < cnt; ++k) {
                const ds_entity_rec& e = E[b0 + k];
                const long long f = worst ? 1024 : uniform_ll(g, a.lo, a.hi);
                const RatT<u128> dur =
                    rat_mul(RatT<u128>{u128(e.exec_num), u128(e.exec_den)}, rat_reduce(u128(f), u128(1024)), ovf);
                if (rat_cmp(dur, window) > 0) window = dur;
            }
        }
        clock = rat_add(clock, window, ovf);
    }
    const RatT<u128> bound{u128(a.bounds[10 * d]), u128(a.bounds[10 * d + 1])};
    const RatT<u128> q = rat_div(clock, bound, ovf);
    ovf |= ((q.n | q.d) >> 64) != 0;
    a.st[t] = ovf ? DS_EOVERFLOW : DS_OK;
    a.over[t] = rat_cmp(clock, bound) > 0;
    // to_double(makespan / bound): both parts to double, one rounded divide
    a.ratio[t] = __ddiv_rn(__ull2double_rn(u64(q.n)), __ull2double_rn(u64(q.d)));
}

}  // namespace ds

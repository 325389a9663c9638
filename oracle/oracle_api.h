/* TEST INFRASTRUCTURE — oracle only (tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs). Never part of the product.
 *
 * One C interface, two implementations:
 *   oracle/_ref/libdagsched_ref.so   the reference's own sources
 *                                    (/root/reference/proj/src/*.cpp) compiled
 *                                    unmodified against oracle/shim/ (prefix ref_)
 *   oracle/_build/libdagsched_oracle.so  the independent restatement in
 *                                    oracle/src/ (prefix orc_)
 * Both speak the packed batch format of include/dagsched_b200.h (ds_dag_batch):
 * per DAG a contiguous node range in id order (local index = rank of the id)
 * and a contiguous edge range of (from << 16) | to local-index pairs.
 *
 * Bounds layout: bounds[d * 10 + 2 * k + {0: num, 1: den}], k in
 * DS_BOUND_{PROPOSED, GREEDY, GREEDY_UNAWARE, GRAHAM_PARA, LOWER}; a bound that
 * was not requested is written as 0/0. Status codes are the DS_* codes.
 */
#ifndef DAGSCHED_ORACLE_API_H
#define DAGSCHED_ORACLE_API_H

#include <stdint.h>

#include "../include/dagsched_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_DECLARE(P)                                                            \
    const char* P##last_error(void);                                                 \
    void P##free(void* p);                                                           \
    /* corpus handle: parsed DagTasks held in the implementation's own types */      \
    void* P##corpus_from_packed(const ds_dag_batch* batch, int64_t min_load_num,     \
                                int64_t min_load_den, int32_t* status);              \
    void* P##corpus_generate(const ds_gen_config* cfg, int64_t count);               \
    int P##corpus_size(void* h, uint64_t* n_dags, uint64_t* n_nodes,                 \
                       uint64_t* n_edges);                                           \
    int P##corpus_pack(void* h, uint32_t* node_off, uint32_t* edge_off,              \
                       int64_t* load_num, int64_t* load_den, uint32_t* edges);       \
    void P##corpus_free(void* h);                                                    \
    /* evaluate_corpus (+ lower_bound) over the handle; returns wall seconds */      \
    double P##corpus_evaluate(void* h, const ds_platform* plat, uint32_t method_mask,\
                              int parallel, int32_t* status, int64_t* bounds);       \
    /* one DAG (index d of the handle) -> JSON text, caller frees with P##free */   \
    char* P##scheme_json(void* h, uint64_t d, const ds_platform* plat);              \
    char* P##analyze_json(void* h, uint64_t d, const ds_platform* plat);

ORACLE_DECLARE(ref_)
ORACLE_DECLARE(orc_)

/* corpus_from_packed with the tasks' real node ids ([N], ascending per DAG);
 * write_scheme then prints ids instead of ranks. ref_ only. */
void* ref_corpus_from_packed_ids(const ds_dag_batch* batch, int64_t min_load_num, int64_t min_load_den,
                                 const int64_t* node_ids, int32_t* status);

/* The reference's run_validation (experiment.cpp:163-240) on
 * generate_corpus(cfg, corpus_size); ref_ only. out = {tasks, runs,
 * violations} and dbl = {mean_tightness_worst, mean_tightness_scaled}. */
int ref_run_validation(const ds_gen_config* cfg, int corpus_size, const ds_platform* plat, int samples,
                       int64_t smin_num, int64_t smin_den, int64_t smax_num, int64_t smax_den, int parallel,
                       int64_t* out, double* dbl);

/* The reference's run_experiment + write_csv (experiment.cpp:81-161): sweep
 * 'M', 'P' or 'V' over values[n_values]; methods as a DS_M_* mask (bits 0-3),
 * normalised to method index `normalize_to`. Returns malloc'd CSV (ref_free)
 * or NULL (ref_last_error). */
char* ref_run_experiment(char sweep, const long long* values, int n_values, const ds_gen_config* base,
                         const ds_platform* plat, int corpus_size, uint32_t methods, int normalize_to);

/* simulate_greedy (simulator.cpp:96-190) per DAG of the handle, `runs` times
 * with policy seed policy_seed + r: status[n*runs], makespan[n*runs*2]. */
int ref_sim_greedy(void* h, const ds_platform* p, int policy, uint64_t policy_seed, int runs, int scaled,
                   uint64_t time_seed, int64_t smin_n, int64_t smin_d, int64_t smax_n, int64_t smax_d,
                   int32_t* status, int64_t* makespan);
/* write_trace(simulate_greedy(...)) / write_trace(simulate_scheme(schedule(...))) for DAG d. */
char* ref_sim_greedy_trace(void* h, uint64_t d, const ds_platform* p, int policy, uint64_t policy_seed, int scaled,
                           uint64_t time_seed, int64_t smin_n, int64_t smin_d, int64_t smax_n, int64_t smax_d);
char* ref_sim_scheme_trace(void* h, uint64_t d, const ds_platform* p, int scaled, uint64_t time_seed,
                           int64_t smin_n, int64_t smin_d, int64_t smax_n, int64_t smax_d);
/* write_task(read_task(json, min_load)) (task_io.cpp:40-91); NULL + *status on failure. */
char* ref_task_roundtrip(const char* json, int64_t min_n, int64_t min_d, int has_seed, uint64_t seed,
                         int32_t* status);
/* write_bench_table(run_benchmarks(...)) (experiment.cpp:242-307). */
char* ref_run_benchmarks(const char* const* paths, int n_paths, const int* sms, int n_sms, const long long* avgs,
                         int n_avgs, int greedy_runs, uint64_t seed);

#undef ORACLE_DECLARE

#ifdef __cplusplus
}
#endif

#endif

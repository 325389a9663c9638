/* dagsched_b200 — C-ABI drop-in boundary for the DAG-scheduler hot path on B200.
 *
 * The reference (arxiv/paper_2602_20826, /root/reference/proj) has no FFI: its
 * boundary is the C++ library API of static lib `dagsched`
 * (proj/include/dagsched/*.hpp). This header is the thin C layer underneath the
 * kept C++ API (include/dagsched/*.hpp in this repo); every entry point names
 * the reference function it replaces.
 *
 * Rules: POD structs only; the caller owns every buffer; no exceptions cross
 * this boundary; every function returns a DS_* status and sets a thread-local
 * message readable with ds_last_error().
 */
#ifndef DAGSCHED_B200_H
#define DAGSCHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ----------------------------------------------------------- status codes */
#define DS_OK 0
#define DS_EINVAL 1      /* std::invalid_argument: bad Platform / GenConfig / args  */
#define DS_EOVERFLOW 3   /* std::overflow_error: exact value outside the ABI range */
#define DS_ECUDA 4       /* CUDA runtime error                                     */
#define DS_EINVARIANT 5  /* std::logic_error: scheduler/simulator invariant broken */
#define DS_ETOOBIG 6     /* DAG larger than DS_MAX_NODES                           */
#define DS_ENOMEM 7
#define DS_ENODEV 8      /* no CUDA device / extension cannot run                  */
/* ValidationError family (dag.cpp:22-138, scheduler.cpp:177-182), one code per
 * message so parity can be checked per DAG. Checked in the reference's order. */
#define DS_E_EMPTY 10      /* "task has no nodes"                         dag.cpp:26  */
#define DS_E_DUP_ID 11     /* "duplicate node id"                         dag.cpp:30-34 */
#define DS_E_LOAD 12       /* "load ... below minimum"                    dag.cpp:35-41 */
#define DS_E_PERIOD 13     /* "period must be positive"                   dag.cpp:42-44 */
#define DS_E_EDGE 14       /* "edge ... references unknown node"          dag.cpp:57-60 */
#define DS_E_SELFLOOP 15   /* "cycle detected: self-loop"                 dag.cpp:61-64 */
#define DS_E_CYCLE 16      /* "cycle detected involving nodes"            dag.cpp:89-95 */
#define DS_E_SOURCES 17    /* "expected a single source node"             dag.cpp:102-105 */
#define DS_E_SINKS 18      /* "expected a single sink node"               dag.cpp:106-108 */
#define DS_E_LOAD_TMIN 19  /* "load below the platform time unit"         scheduler.cpp:177-182 */

/* Largest DAG the device path accepts. Size classes: n <= 64 one warp per
 * DAG with 1-word masks (k1_fast / k1_front / k1_analyse<1>), <= 256 four
 * words (k1_analyse<4>), <= 512 eight words in 191 KB of shared memory and
 * <= 1024 sixteen words in a global-memory warp state (k1_big). */
#define DS_MAX_NODES 1024

/* Bound slots / method mask bits. Methods mirror experiment.hpp:14
 * (Method::{proposed, greedy, greedy_unaware, graham_para}); LOWER is
 * lower_bound (analysis.cpp:72-81). */
#define DS_BOUND_PROPOSED 0
#define DS_BOUND_GREEDY 1
#define DS_BOUND_GREEDY_UNAWARE 2
#define DS_BOUND_GRAHAM_PARA 3
#define DS_BOUND_LOWER 4
#define DS_N_BOUNDS 5
#define DS_M_PROPOSED (1u << DS_BOUND_PROPOSED)
#define DS_M_GREEDY (1u << DS_BOUND_GREEDY)
#define DS_M_GREEDY_UNAWARE (1u << DS_BOUND_GREEDY_UNAWARE)
#define DS_M_GRAHAM_PARA (1u << DS_BOUND_GRAHAM_PARA)
#define DS_M_LOWER (1u << DS_BOUND_LOWER)
#define DS_M_ALL 0x1fu

/* Flags for the batch entry points. */
#define DS_F_DEVICE_PTRS 1u /* batch and result pointers are device memory on `device` */
#define DS_F_PINNED 2u      /* (corpus generation) allocate host arrays pinned         */
#define DS_F_GPU_GENERATE 4u /* (corpus generation) generate on the calling thread's
                              * current CUDA device (K5), copy into the host arrays  */

/* --------------------------------------------------------------- inputs */
/* Platform (exec_model.hpp:11-19): M identical SMs and the time floor t_min,
 * plus how the device applies DagTask::make's load floor (dag.cpp:35-41) to a
 * packed batch. `flags` = 0: min_load = t_min (generate() makes its tasks
 * that way, generator.cpp:94-95); DS_PF_MIN_LOAD_ONE: min_load = 1 (the
 * default argument of DagTask::make, dag.hpp:38-41); DS_PF_PREMADE: the tasks
 * were already made on the host (the kept C++ API), only load > 0 is checked.
 * Independently of the floor, a load below t_min fails only the proposed
 * method, with DS_E_LOAD_TMIN (schedule()'s own check, scheduler.cpp:177-182);
 * the other bounds are computed as the reference computes them. */
#define DS_PF_MIN_LOAD_ONE 1
#define DS_PF_PREMADE 2
typedef struct ds_platform {
    int32_t sm_count;
    int32_t flags;
    int64_t tmin_num;
    int64_t tmin_den;
} ds_platform;

/* Packed batch of DAGs (the batch form of std::vector<DagTask>).
 * DAG d owns nodes [node_off[d], node_off[d+1]) in ascending-id order — the
 * local index of a node is the rank of its id, which is how every "ties by
 * id" rule of the reference is preserved — and edges
 * [edge_off[d], edge_off[d+1]), each packed as (from_local << 16) | to_local.
 * Loads are exact rationals load_num/load_den (den > 0, need not be reduced);
 * load_den == NULL means every denominator is 1. Array indices are relative
 * to the first offset: node i of the batch is load_num[i - node_off[0]], so a
 * sub-batch is just shifted pointers (see ds_analyze_batch_multi). */
typedef struct ds_dag_batch {
    uint64_t n_dags;
    const uint32_t* node_off; /* [n_dags + 1] */
    const uint32_t* edge_off; /* [n_dags + 1] */
    const int64_t* load_num;  /* [node_off[n_dags]] */
    const int64_t* load_den;  /* [node_off[n_dags]] or NULL */
    const uint32_t* edges;    /* [edge_off[n_dags]] */
} ds_dag_batch;

/* Compact wire form of a batch with integer loads in [1, 65535] and at most
 * 256 nodes per DAG (every GenConfig corpus with integer loads, e.g. C5): the
 * same offsets, 16-bit loads and 16-bit edges (from << 8 | to). 2.4x fewer
 * bytes over PCIe than ds_dag_batch (C5: 199 MB instead of 488 MB per 1M
 * DAGs); the device widens it before the analysis. */
typedef struct ds_dag_batch16 {
    uint64_t n_dags;
    const uint32_t* node_off; /* [n_dags + 1] */
    const uint32_t* edge_off; /* [n_dags + 1] */
    const uint16_t* load;     /* [node_off[n_dags]] integer load num (den 1)    */
    const uint16_t* edges;    /* [edge_off[n_dags]] from << 8 | to              */
} ds_dag_batch16;

/* Triangular wire form of a batch whose local node indices are a topological
 * order (every edge u < v), with at most 64 nodes per DAG and 16-bit integer
 * loads: instead of an edge list, each DAG carries its strictly lower
 * triangular adjacency matrix as bits — the predecessors of node v (v = 1 ..
 * n-1) are bits [v(v-1)/2, v(v-1)/2 + v) of the DAG's words, bit
 * v(v-1)/2 + u set iff (u, v) is an edge; little-endian within u32 words.
 * DAG d's words are adj[adj_off[d] - adj_off[0] .. adj_off[d+1] - adj_off[0])
 * (any number >= ceil(n(n-1)/64) words). Duplicate edges are impossible and
 * order is implied. C5: ~107 B per DAG over PCIe instead of 199 B
 * (ds_dag_batch16) or 488 B (ds_dag_batch); the device expands it. */
typedef struct ds_dag_batch_tri {
    uint64_t n_dags;
    const uint32_t* node_off; /* [n_dags + 1] */
    const uint32_t* adj_off;  /* [n_dags + 1] in u32 words */
    const uint16_t* load;     /* [node_off[n_dags]] integer load num (den 1)    */
    const uint32_t* adj;      /* [adj_off[n_dags]] adjacency bit matrices       */
} ds_dag_batch_tri;

/* Per-DAG results of the batched analysis (evaluate_corpus + lower_bound). */
typedef struct ds_results {
    int32_t* status;   /* [n_dags] DS_OK or a per-DAG DS_E* / DS_EOVERFLOW code   */
    int64_t* bounds;   /* [n_dags * 10]: bound k at (2k, 2k+1) = (num, den), reduced,
                          den > 0; 0/0 when the method bit was not requested       */
    uint16_t* n_groups;/* optional [n_dags]: executed balanced groups (may be NULL) */
} ds_results;

/* GenConfig (generator.hpp:15-28). */
typedef struct ds_gen_config {
    int32_t depth_min, depth_max, max_width, integer_loads;
    int64_t avg_load_num, avg_load_den;
    double load_jitter, edge_density;
    uint64_t seed;
    int64_t tmin_num, tmin_den;
    int32_t exact_mean, reserved;
} ds_gen_config;

/* ------------------------------------------------- schedule detail output */
/* EntityRecord (scheduler.hpp:31-39) minus preds, in creation order: for each
 * executed group its launches (launch order) then its members (id order). */
typedef struct ds_entity_rec {
    uint16_t origin;      /* local node index (EntityId::origin)                 */
    uint16_t generation;  /* EntityId::generation                                */
    uint8_t part;         /* 0 whole, 1 parallel, 2 residual (EntityId::Part)    */
    uint8_t launched;     /* EntityRecord::launched                              */
    uint16_t group;       /* executed-group index                                */
    int32_t parallelism;  /* SMs held                                            */
    int32_t reserved;
    int64_t load_num, load_den;  /* EntityRecord::load                           */
    int64_t exec_num, exec_den;  /* EntityRecord::exec (= duration for launches) */
    int64_t res_num, res_den;    /* parallel segments: residual load left behind  */
} ds_entity_rec;

/* GroupPlan (scheduler.hpp:56-64) plus what is needed to materialise the
 * augmented graph (extra deps) on the host. */
typedef struct ds_group_rec {
    int64_t resp_num, resp_den;  /* GroupPlan::response                          */
    int32_t spare_sms;           /* GroupPlan::spare_sms                         */
    uint16_t div_group;          /* index of the division group it executes      */
    uint16_t bottleneck;         /* entity index (within the DAG) of v_R         */
    uint16_t first_entity;       /* launches then members, contiguous            */
    uint16_t n_launches;
    uint16_t n_members;
    uint16_t reserved;
} ds_group_rec;

/* Capacities: entities per DAG <= 2 n, executed groups per DAG <= n. Slot bases
 * are 2*node_off[d] for entities and node_off[d] for groups. */
typedef struct ds_scheme_out {
    int32_t* status;          /* [n_dags]                                        */
    uint16_t* n_entities;     /* [n_dags]                                        */
    uint16_t* n_groups;       /* [n_dags]                                        */
    uint16_t* n_div_groups;   /* [n_dags] size of the division Π                 */
    int16_t* node_block;      /* [N] block index of each node (build_blocks)     */
    int16_t* node_div_group;  /* [N] division group of each node (build_groups)  */
    ds_entity_rec* entities;  /* [2N]                                            */
    ds_group_rec* groups;     /* [N]                                             */
    int64_t* bounds;          /* [n_dags * 10] as in ds_results                  */
    uint64_t* unlaunched;     /* per executed group, the node mask of candidates
                                 not launched whole (they get the extra dep
                                 v_R -> candidate): DAG d (n nodes, w =
                                 ceil(n/64) words per mask) group g at
                                 unlaunched[u_d + g*w .. + w), u_d = the sum
                                 over earlier DAGs k of n_k * w_k (0 when
                                 NULL: not returned)                          */
} ds_scheme_out;

/* ------------------------------------------------------ executor (K2/K3) */
/* Node workloads (K2). Every entity of a schedule is one launch of one of
 * these memory-bound kernels over its element range of its node's buffers;
 * per-CTA start/end are stamped with %globaltimer and %smid. */
#define DS_WL_MIX32 0   /* y[i] = mix(x[i]), uint32, LDG.128/STG.128: 8 B/elem   */
#define DS_WL_AXPY32 1  /* y[i] = a*x[i] + y[i], fp32 (no FMA contraction): 12 B  */
/* (2: retired — an older 4 x 24 KB bulk-copy ring, superseded by 3)       */
#define DS_WL_MIX32_TMA 3  /* DS_WL_MIX32 through a warp-specialised 6 x 32 KB
                              cp.async.bulk ring (1 producer + 16 consumer
                              warps, 544 threads per CTA): 8 B/elem            */
#define DS_WL_MIX32_LDG8 4 /* DS_WL_MIX32 with 8 LDG.128 in flight per thread  */
#define DS_WL_LAST 4

/* One schedulable entity (EntityRecord, scheduler.hpp:31-39) as executed:
 * grid = parallelism CTAs, one CTA per SM enforced by the kernel's shared
 * memory footprint; elements [elem_lo, elem_hi) of node `node`'s buffers. */
typedef struct ds_exec_entity {
    int32_t group;        /* executed group, -1 when the plan has no groups    */
    int32_t parallelism;  /* CTAs = SMs held                                   */
    int32_t node;         /* origin node (buffer)                              */
    uint32_t pred_off;    /* preds[pred_off .. pred_off + n_preds)             */
    uint32_t n_preds;
    uint32_t reserved;
    uint64_t elem_lo, elem_hi;
} ds_exec_entity;

typedef struct ds_exec_plan {
    int32_t n_entities;
    int32_t n_nodes;
    const ds_exec_entity* entities;
    const uint32_t* preds;       /* entity indices (graph edges pred -> entity)  */
    const uint64_t* node_elems;  /* [n_nodes] buffer length per node             */
    int32_t barrier_groups;      /* DS_PLAN_*: how groups are ordered             */
    int32_t reserved;
} ds_exec_plan;

/* ds_exec_plan.barrier_groups. DEPS: only the plan's edges order entities
 * (the augmented graph: original edges + extra dependencies Ē). BARRIERS:
 * group g+1 starts after all of group g (simulate_scheme semantics,
 * simulator.cpp:44-94). PRIORITY (DS_ENGINE_DYNAMIC or DS_ENGINE_GRAPH): the plan's edges
 * are the precedence edges alone (original edges resolved to segment chains,
 * no Ē) and the engine enforces the group order itself — no rank of a
 * group-(g+1) entity is claimed while a group-g entity still has unclaimed
 * ranks — so a group's entities always find their quota of SMs free, every
 * group ends within its response after the previous group's last rank (the
 * Theorem-1 induction), and SMs that finish early take the next group's
 * ranks instead of idling behind Ē. On DS_ENGINE_GRAPH the same order is
 * requested from the hardware: each kernel node carries the launch priority
 * of its group (group 0 highest, the last group lowest, the groups spread
 * evenly over the device's priority levels) and the graph is instantiated with
 * cudaGraphInstantiateFlagUseNodePriority, so a freed SM takes a pending CTA
 * of the earliest ready group — best effort (the dispatcher's order, not a
 * device-side claim), checked against the bound per replay like every
 * variant. */
#define DS_PLAN_DEPS 0
#define DS_PLAN_BARRIERS 1
#define DS_PLAN_PRIORITY 2

typedef struct ds_exec_cfg {
    int32_t workload;       /* DS_WL_*                                           */
    int32_t block_threads;  /* threads per CTA (<= 1024)                         */
    uint32_t seed;          /* input initialisation                              */
    int32_t sm_limit;       /* 0: whole GPU; else run inside a green context of
                               this many SMs (multiple of 8 on sm_90+) — an
                               M-SM device for the paper's contended regime   */
    int32_t engine;         /* DS_ENGINE_*                                       */
    int32_t chunk_elems;    /* DS_ENGINE_DYNAMIC: 0 = rank r of an m-rank entity
                               processes the fixed slice r/m; > 0 = its ranks
                               claim chunks of this many elements from the
                               entity's range until it is done (still at most
                               m SMs at a time; late ranks take less)         */
} ds_exec_cfg;

/* Executor engines. GRAPH: one CUDA Graph kernel node per entity (plans
 * DS_PLAN_DEPS / DS_PLAN_BARRIERS / DS_PLAN_PRIORITY). (1 and 4 are retired engines: a static
 * list-scheduled persistent kernel and a ring-streaming variant of DYNAMIC,
 * both measured slower than DYNAMIC.) */
#define DS_ENGINE_GRAPH 0
/* GRAPH_FREE: the graph engine with the launch shape a developer would use
 * without quota control — 4 x parallelism CTAs of 256 threads, no shared
 * memory — so concurrent kernels share SMs and interfere (the naive
 * multi-stream baseline of PAPER.md:533 on real hardware). Stamps then hold
 * 4 x parallelism CTAs per entity. */
#define DS_ENGINE_GRAPH_FREE 2
#define DS_FREE_CTA_FACTOR 4
/* DYNAMIC: one resident CTA per SM, work-conserving: an entity enters a
 * device-side ready queue (plan order = schedule priority) when its last
 * predecessor completes, and idle CTAs claim its m ranks, so it never holds
 * more than its quota of SMs. Any topologically ordered plan (for
 * DS_PLAN_PRIORITY the exact device-side claim order); workloads DS_WL_MIX32 and DS_WL_MIX32_TMA. */
#define DS_ENGINE_DYNAMIC 3
/* STREAMS: no graph — every replay the host launches each entity's kernel on
 * its own stream after cudaStreamWaitEvent on its predecessors' events (and,
 * with group barriers, on the previous group's): naive multi-stream launch as
 * an application writes it. */
#define DS_ENGINE_STREAMS 5

/* Per-replay device-timed spans and, for every replay, per-CTA stamps. */
typedef struct ds_exec_trace {
    uint64_t* span;    /* [replays * 2] min CTA start, max CTA end (ns, %globaltimer) */
    uint64_t* stamps;  /* [replays * total_ctas * 2] start, end per CTA (optional)   */
    uint32_t* smids;   /* [replays * total_ctas] (optional)                          */
    float* launch_ms;  /* [replays] host-side graph launch -> completion, CUDA events */
} ds_exec_trace;

/* ------------------------------------------------------------- functions */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
const char* ds_last_error(void);
const char* ds_version(void);
int ds_device_count(int* count);
/* Page-locked host memory for the batch entry points' arrays (their copies
 * then run at full PCIe rate and asynchronously): cudaMallocHost / cudaFreeHost.
 * No reference equivalent (the reference has no device). */
int ds_pinned_alloc(size_t bytes, void** out);
int ds_pinned_free(void* p);

/* Batched bound analysis — replaces evaluate_corpus (experiment.cpp:52-79 with
 * method_bound :27-39) plus lower_bound (analysis.cpp:72-81). One warp per DAG.
 * Host pointers (pinned or pageable) unless DS_F_DEVICE_PTRS; `stream` is a
 * cudaStream_t (NULL = a library stream). Synchronous for host pointers,
 * asynchronous on `stream` for device pointers. */
int ds_analyze_batch(const ds_dag_batch* batch, const ds_platform* platform,
                     uint32_t method_mask, ds_results* out, int device, void* stream,
                     uint32_t flags);

/* ds_analyze_batch over the compact wire form (host pointers only, pinned
 * for full PCIe speed); results identical to ds_analyze_batch on the same
 * DAGs. A load of 0 is rejected per DAG as in the wide form. */
int ds_analyze_batch16(const ds_dag_batch16* batch, const ds_platform* platform,
                       uint32_t method_mask, ds_results* out, int device);

/* ds_analyze_batch over the triangular wire form (host pointers, pinned for
 * full PCIe speed); results identical to ds_analyze_batch on the same DAGs.
 * A DAG with more than 64 nodes is DS_ETOOBIG in this form. */
int ds_analyze_batch_tri(const ds_dag_batch_tri* batch, const ds_platform* platform,
                         uint32_t method_mask, ds_results* out, int device);

/* Same, sharded as contiguous DAG ranges over `devices` (one host thread per
 * device, no collective), host pointers only; results land in DAG order. */
int ds_analyze_batch_multi(const ds_dag_batch* batch, const ds_platform* platform,
                           uint32_t method_mask, ds_results* out, const int* devices,
                           int n_devices);

/* ds_analyze_batch16 sharded the same way (the compact wire form: 2.4x fewer
 * PCIe bytes per device). */
int ds_analyze_batch16_multi(const ds_dag_batch16* batch, const ds_platform* platform,
                             uint32_t method_mask, ds_results* out, const int* devices,
                             int n_devices);

/* ds_analyze_batch_tri sharded the same way. */
int ds_analyze_batch_tri_multi(const ds_dag_batch_tri* batch, const ds_platform* platform,
                               uint32_t method_mask, ds_results* out, const int* devices,
                               int n_devices);

/* The split both multi entry points use: shard i of n_shards owns DAGs
 * [lo, hi) = [n*i/n_shards, n*(i+1)/n_shards) — the contiguous split of the
 * reference's OpenMP loop over independent DAGs (experiment.cpp:56-66), and
 * the per-rank shard of bench.py / shard.py. Host-only, no device needed. */
int ds_shard_range(uint64_t n_dags, int n_shards, int shard, uint64_t* lo, uint64_t* hi);

/* Full schedule detail — replaces schedule() (scheduler.cpp:175-427) and
 * build_blocks/build_groups (division.cpp:10-126) for a batch; host pointers. */
int ds_schedule_batch(const ds_dag_batch* batch, const ds_platform* platform,
                      ds_scheme_out* out, int device);

/* ------------------------------------------------ greedy simulation (K6) */
/* simulate_greedy (simulator.cpp:96-190) for every DAG of a batch, `runs`
 * times each: run r dispatches with DispatchPolicy `policy` (0 fifo, 1 random)
 * seeded policy_seed + r (run_benchmarks' convention, experiment.cpp:271-276);
 * durations are exec_time(load, min(m^max, M)) times the TimeModel factor
 * (scaled: uniform on the 1/1024 grid of [scale_min, scale_max], generator
 * seeded time_seed, identical for every run). */
typedef struct ds_greedy_cfg {
    int32_t policy;
    int32_t runs;
    uint64_t policy_seed;
    int32_t scaled;   /* TimeModel::Kind: 0 worst_case, 1 scaled */
    int32_t reserved;
    uint64_t time_seed;
    int64_t scale_min_num, scale_min_den, scale_max_num, scale_max_den;
} ds_greedy_cfg;

/* Host pointers. status[n*runs], makespan[n*runs*2] (num, den); events
 * (optional, NULL to skip) [N*runs*4]: per node and run start num/den, finish
 * num/den (index (node_off[d] - node_off[0] + v) * runs + r). Exact rationals
 * (64-bit words, 128-bit redo on overflow); DS_EOVERFLOW where a value leaves
 * int64. DAGs must satisfy DagTask::make (one source; edges as in the batch
 * format, duplicates collapse). */
int ds_simulate_greedy_batch(const ds_dag_batch* batch, const ds_platform* platform,
                             const ds_greedy_cfg* cfg, int32_t* status, int64_t* makespan,
                             int64_t* events, int device);

/* Corpus generation — replaces generate_corpus (generator.cpp:98-108) with
 * identical RNG call order: on the host, parallel over seeds, or with
 * DS_F_GPU_GENERATE on the device (one thread per DAG, K5). The handle owns
 * packed host arrays (pinned when DS_F_PINNED) exposed through ds_corpus_view. */
int ds_corpus_generate(const ds_gen_config* cfg, int64_t count, uint32_t flags,
                       void** handle);
int ds_corpus_view(void* handle, ds_dag_batch* view);
/* Device milliseconds of a DS_F_GPU_GENERATE generation (kernels + scans; 0
 * for host generation). */
float ds_corpus_gen_ms(void* handle);
void ds_corpus_free(void* handle);

/* Timed-analysis session: uploads a batch once and replays the kernel on it
 * (bench.py's device-resident `value` leg). */
int ds_session_create(const ds_dag_batch* batch, const ds_platform* platform,
                      uint32_t method_mask, int device, void** session);
/* Launches the analysis kernel on the session's stream; returns the kernel's
 * duration in ms measured with CUDA events on that stream. */
int ds_session_run(void* session, float* kernel_ms);
/* Per-kernel device times of the last run (CUDA events between consecutive
 * launches on the session's stream): fills up to `max` entries of ms[] and
 * names[] (static strings), returns the count, or -status on error. */
int ds_session_kernel_times(void* session, float* ms, const char** names, int max);
/* Copies results of the last run back to host buffers. */
int ds_session_results(void* session, ds_results* out);
int ds_session_free(void* session);

/* Theorem-1 validation — replaces run_validation (experiment.cpp:163-240)
 * over a given batch: per DAG the proposed schedule (K1) is simulated at
 * worst case and `samples` times with durations scaled by factors k/1024,
 * k ~ uniform_int_distribution<long long>(ceil(smin*1024), floor(smax*1024))
 * over std::mt19937_64(seed + 7919*d + s) — bit-exact with the reference
 * (simulator.cpp:14-94). Per-DAG arrays are optional (NULL to skip). */
typedef struct ds_validation {
    int64_t tasks, runs, violations;
    double mean_tightness_worst, mean_tightness_scaled;
} ds_validation;
int ds_validate_batch(const ds_dag_batch* batch, const ds_platform* platform, int samples, int64_t smin_num,
                      int64_t smin_den, int64_t smax_num, int64_t smax_den, uint64_t seed, int32_t* status,
                      int32_t* violations, double* tight_worst, double* tight_scaled, ds_validation* summary,
                      int device);

/* Executor (K3) — replaces simulate_scheme (simulator.cpp:44-94) with real
 * execution: builds device buffers (inputs initialised from cfg->seed) and a
 * CUDA Graph with one kernel node per entity (grid = quota) and an edge per
 * entry of preds (plus group barriers when plan->barrier_groups). */
int ds_exec_create(const ds_exec_plan* plan, const ds_exec_cfg* cfg, int device, void** exec);
/* Replays the graph `replays` times (after `warmup` untimed replays that are
 * not recorded); fills the trace arrays for the recorded replays. */
int ds_exec_run(void* exec, int warmup, int replays, ds_exec_trace* trace);
/* Total CTAs of one replay (sum of parallelism) — sizes the stamp arrays. */
int ds_exec_total_ctas(void* exec, uint64_t* total);
/* SMs the executor runs on (the green-context size when sm_limit > 0). */
int ds_exec_sm_count(void* exec, int* sms);
/* Copies node `node`'s output buffer (uint32 / fp32 words) to host memory. */
int ds_exec_read_output(void* exec, int node, void* host, uint64_t n_elems);
int ds_exec_free(void* exec);

/* Node-kernel roofline probe: one launch of `workload` over ctas CTAs x
 * elems_per_cta elements (1 CTA per SM), timed with CUDA events over `reps`
 * launches after warm-up; returns the mean ms per launch and the per-CTA
 * globaltimer span of the last launch. */
int ds_node_kernel_bench(int workload, int ctas, uint64_t elems_per_cta, int block_threads, int reps,
                         float* ms_per_launch, uint64_t* span_ns, int device);
/* Placement probe (diagnostic): one CTA per SM; the SMs whose %smid bit is set
 * in mask8 (8 x 32 bits) each stream `elems` uint32 through the mix kernel;
 * *avg_span_ns = mean device span over `reps` launches (HBM-resident data). */
int ds_node_placement_bench(const uint32_t* mask8, uint64_t elems, int reps, double* avg_span_ns, int device);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* DAGSCHED_B200_H */

// TEST INFRASTRUCTURE — oracle only.
//
// C wrapper (prefix ref_) around the reference library compiled from
// /root/reference/proj/src/*.cpp against oracle/shim/. Everything below calls
// the reference's own public API (proj/include/dagsched/*.hpp): DagTask::make,
// generate_corpus, evaluate_corpus, lower_bound, schedule, analyze,
// write_scheme. It only translates the packed batch format and maps the
// reference's exceptions to DS_* status codes.
#include "dagsched/analysis.hpp"
#include "dagsched/experiment.hpp"
#include "dagsched/generator.hpp"
#include "dagsched/scheduler.hpp"
#include "dagsched/task_io.hpp"

#include "oracle_api.h"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

using namespace dagsched;

namespace {

thread_local std::string g_err;

int status_of_validation(const std::string& m) {
    auto has = [&](const char* s) { return m.find(s) != std::string::npos; };
    if (has("no nodes")) return DS_E_EMPTY;
    if (has("duplicate node id")) return DS_E_DUP_ID;
    if (has("below the platform time unit")) return DS_E_LOAD_TMIN;
    if (has("below minimum")) return DS_E_LOAD;
    if (has("period")) return DS_E_PERIOD;
    if (has("unknown node")) return DS_E_EDGE;
    if (has("self-loop")) return DS_E_SELFLOOP;
    if (has("cycle detected")) return DS_E_CYCLE;
    if (has("single source")) return DS_E_SOURCES;
    if (has("single sink")) return DS_E_SINKS;
    return DS_EINVAL;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return DS_OK;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return status_of_validation(e.what());
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return DS_EOVERFLOW;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return DS_EINVAL;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return DS_EINVAL;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return DS_EINVARIANT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return DS_EINVAL;
    }
}

struct Corpus {
    std::vector<DagTask> tasks;
    std::vector<std::size_t> index;  // batch index of each parsed task
    std::uint64_t n_dags = 0;
};

Rational rat(int64_t n, int64_t d) { return Rational(BigInt(n), BigInt(d)); }

Platform platform_of(const ds_platform* p) {
    return Platform{p->sm_count, rat(p->tmin_num, p->tmin_den)};
}

bool to_i64(const BigInt& v, int64_t& out) {
    if (v > BigInt(INT64_MAX) || v < BigInt(INT64_MIN)) return false;
    out = static_cast<int64_t>(v.convert_to<long long>());
    return true;
}

bool put(const Rational& r, int64_t* slot) {
    return to_i64(numerator(r), slot[0]) && to_i64(denominator(r), slot[1]);
}

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

void* ref_corpus_from_packed(const ds_dag_batch* b, int64_t min_num, int64_t min_den,
                             int32_t* status) {
    auto c = std::make_unique<Corpus>();
    c->n_dags = b->n_dags;
    c->tasks.reserve(b->n_dags);
    for (std::uint64_t d = 0; d < b->n_dags; ++d) {
        std::vector<DagNode> nodes;
        std::vector<std::pair<NodeId, NodeId>> edges;
        for (uint32_t i = b->node_off[d]; i < b->node_off[d + 1]; ++i) {
            int64_t den = b->load_den ? b->load_den[i - b->node_off[0]] : 1;
            nodes.push_back(DagNode{i - b->node_off[d], rat(b->load_num[i - b->node_off[0]], den)});
        }
        for (uint32_t e = b->edge_off[d]; e < b->edge_off[d + 1]; ++e) {
            edges.emplace_back(b->edges[e - b->edge_off[0]] >> 16, b->edges[e - b->edge_off[0]] & 0xffffu);
        }
        int st = guarded([&] {
            c->tasks.push_back(DagTask::make(std::move(nodes), std::move(edges),
                                             std::nullopt, rat(min_num, min_den)));
            c->index.push_back(d);
        });
        if (status) status[d] = st;
    }
    return c.release();
}

// The same with the tasks' real node ids (node_ids[i - node_off[0]] for node
// i of the batch, ascending within a DAG; a local index >= n, the packer's
// "unknown endpoint", maps to an id above every node's) so write_scheme
// prints ids, as the reference does for a task read from JSON.
void* ref_corpus_from_packed_ids(const ds_dag_batch* b, int64_t min_num, int64_t min_den,
                                 const int64_t* node_ids, int32_t* status) {
    auto c = std::make_unique<Corpus>();
    c->n_dags = b->n_dags;
    c->tasks.reserve(b->n_dags);
    for (std::uint64_t d = 0; d < b->n_dags; ++d) {
        std::vector<DagNode> nodes;
        std::vector<std::pair<NodeId, NodeId>> edges;
        const uint32_t n0 = b->node_off[d] - b->node_off[0], n = b->node_off[d + 1] - b->node_off[d];
        NodeId top = 0;
        for (uint32_t k = 0; k < n; ++k) top = std::max<NodeId>(top, NodeId(node_ids[n0 + k]));
        auto id_of = [&](uint32_t k) { return k < n ? NodeId(node_ids[n0 + k]) : NodeId(top + 1 + (k - n)); };
        for (uint32_t k = 0; k < n; ++k) {
            int64_t den = b->load_den ? b->load_den[n0 + k] : 1;
            nodes.push_back(DagNode{id_of(k), rat(b->load_num[n0 + k], den)});
        }
        for (uint32_t e = b->edge_off[d]; e < b->edge_off[d + 1]; ++e) {
            const uint32_t w = b->edges[e - b->edge_off[0]];
            edges.emplace_back(id_of(w >> 16), id_of(w & 0xffffu));
        }
        int st = guarded([&] {
            c->tasks.push_back(DagTask::make(std::move(nodes), std::move(edges),
                                             std::nullopt, rat(min_num, min_den)));
            c->index.push_back(d);
        });
        if (status) status[d] = st;
    }
    return c.release();
}

void* ref_corpus_generate(const ds_gen_config* g, int64_t count) {
    Corpus* out = nullptr;
    int st = guarded([&] {
        GenConfig cfg;
        cfg.depth_min = g->depth_min;
        cfg.depth_max = g->depth_max;
        cfg.max_width = g->max_width;
        cfg.avg_load = rat(g->avg_load_num, g->avg_load_den);
        cfg.load_jitter = g->load_jitter;
        cfg.edge_density = g->edge_density;
        cfg.seed = g->seed;
        cfg.integer_loads = g->integer_loads != 0;
        cfg.exact_mean = g->exact_mean != 0;
        cfg.t_min = rat(g->tmin_num, g->tmin_den);
        auto c = std::make_unique<Corpus>();
        c->tasks = generate_corpus(cfg, static_cast<int>(count));
        c->n_dags = c->tasks.size();
        for (std::size_t i = 0; i < c->tasks.size(); ++i) c->index.push_back(i);
        out = c.release();
    });
    return st == DS_OK ? out : nullptr;
}

int ref_corpus_size(void* h, uint64_t* n_dags, uint64_t* n_nodes, uint64_t* n_edges) {
    auto* c = static_cast<Corpus*>(h);
    uint64_t nn = 0, ne = 0;
    for (const DagTask& t : c->tasks) {
        nn += t.size();
        ne += t.edges().size();
    }
    *n_dags = c->tasks.size();
    *n_nodes = nn;
    *n_edges = ne;
    return DS_OK;
}

int ref_corpus_pack(void* h, uint32_t* node_off, uint32_t* edge_off, int64_t* load_num,
                    int64_t* load_den, uint32_t* edges) {
    auto* c = static_cast<Corpus*>(h);
    uint32_t no = 0, eo = 0;
    for (std::size_t d = 0; d < c->tasks.size(); ++d) {
        const DagTask& t = c->tasks[d];
        node_off[d] = no;
        edge_off[d] = eo;
        std::vector<NodeId> ids;
        for (const DagNode& n : t.nodes()) {
            if (!to_i64(numerator(n.load), load_num[no]) ||
                !to_i64(denominator(n.load), load_den[no])) {
                g_err = "load outside int64";
                return DS_EOVERFLOW;
            }
            ids.push_back(n.id);
            ++no;
        }
        auto local = [&](NodeId id) {
            return static_cast<uint32_t>(std::lower_bound(ids.begin(), ids.end(), id) -
                                         ids.begin());
        };
        for (const auto& [u, v] : t.edges()) edges[eo++] = (local(u) << 16) | local(v);
    }
    node_off[c->tasks.size()] = no;
    edge_off[c->tasks.size()] = eo;
    return DS_OK;
}

void ref_corpus_free(void* h) { delete static_cast<Corpus*>(h); }

double ref_corpus_evaluate(void* h, const ds_platform* p, uint32_t mask, int parallel,
                           int32_t* status, int64_t* bounds) {
    auto* c = static_cast<Corpus*>(h);
    Platform plat = platform_of(p);
    std::vector<Method> methods;
    std::vector<int> slot;
    const Method all[4] = {Method::proposed, Method::greedy, Method::greedy_unaware,
                           Method::graham_para};
    for (int k = 0; k < 4; ++k) {
        if (mask & (1u << k)) {
            methods.push_back(all[k]);
            slot.push_back(k);
        }
    }
    std::vector<std::vector<Rational>> rows;
    std::vector<Rational> lowers(c->tasks.size());
    auto t0 = std::chrono::steady_clock::now();
    int st = guarded([&] {
        // The reference's own batch entry point (experiment.cpp:52-79).
        rows = evaluate_corpus(c->tasks, plat, methods, parallel != 0);
        if (mask & DS_M_LOWER) {
            if (parallel) {
#pragma omp parallel for schedule(dynamic)
                for (long long i = 0; i < static_cast<long long>(c->tasks.size()); ++i) {
                    lowers[i] = lower_bound(c->tasks[i], plat);
                }
            } else {
                for (std::size_t i = 0; i < c->tasks.size(); ++i) {
                    lowers[i] = lower_bound(c->tasks[i], plat);
                }
            }
        }
    });
    auto t1 = std::chrono::steady_clock::now();
    if (st != DS_OK) {
        // An exception escaped the batch: redo per task to attribute it.
        rows.assign(c->tasks.size(), {});
        for (std::size_t i = 0; i < c->tasks.size(); ++i) {
            int s = guarded([&] {
                rows[i] = evaluate_corpus({c->tasks[i]}, plat, methods, false)[0];
                if (mask & DS_M_LOWER) lowers[i] = lower_bound(c->tasks[i], plat);
            });
            if (s != DS_OK) rows[i].clear();
            if (status) status[c->index[i]] = s;
        }
    }
    for (std::size_t i = 0; i < c->tasks.size(); ++i) {
        std::size_t d = c->index[i];
        int64_t* b = bounds + d * 10;
        for (int k = 0; k < 10; ++k) b[k] = 0;
        if (st != DS_OK && status && status[d] != DS_OK) continue;
        bool ok = true;
        for (std::size_t m = 0; m < methods.size(); ++m) ok &= put(rows[i][m], b + 2 * slot[m]);
        if (mask & DS_M_LOWER) ok &= put(lowers[i], b + 2 * DS_BOUND_LOWER);
        if (!ok) for (int k = 0; k < 10; ++k) b[k] = 0;  // failed DAGs carry no bounds
        if (status) status[d] = ok ? DS_OK : DS_EOVERFLOW;
    }
    return std::chrono::duration<double>(t1 - t0).count();
}

char* ref_scheme_json(void* h, uint64_t d, const ds_platform* p) {
    auto* c = static_cast<Corpus*>(h);
    std::string text;
    int st = guarded([&] {
        std::ostringstream out;
        write_scheme(schedule(c->tasks.at(d), platform_of(p)), out);
        text = out.str();
    });
    return st == DS_OK ? dup(text) : nullptr;
}

char* ref_analyze_json(void* h, uint64_t d, const ds_platform* p) {
    auto* c = static_cast<Corpus*>(h);
    std::string text;
    int st = guarded([&] {
        MakespanReport r = analyze(c->tasks.at(d), platform_of(p));
        std::ostringstream out;
        out << "{\"per_group_response\": [";
        for (std::size_t i = 0; i < r.per_group_response.size(); ++i) {
            out << (i ? ", " : "") << '"' << format_exact(r.per_group_response[i]) << '"';
        }
        out << "], \"proposed\": \"" << format_exact(r.proposed) << "\", \"greedy\": \""
            << format_exact(r.greedy) << "\", \"greedy_unaware\": \""
            << format_exact(r.greedy_unaware) << "\", \"graham_para\": \""
            << format_exact(r.graham_para) << "\", \"lower\": \"" << format_exact(r.lower)
            << "\", \"normalized\": {";
        bool first = true;
        for (const auto& [k, v] : r.normalized) {
            out << (first ? "" : ", ") << '"' << k << "\": \"" << format_exact(v) << '"';
            first = false;
        }
        out << "}}";
        text = out.str();
    });
    return st == DS_OK ? dup(text) : nullptr;
}

}  // extern "C"

extern "C" int ref_run_validation(const ds_gen_config* g, int corpus_size, const ds_platform* p, int samples,
                                  int64_t smin_num, int64_t smin_den, int64_t smax_num, int64_t smax_den,
                                  int parallel, int64_t* out, double* dbl) {
    return guarded([&] {
        GenConfig cfg;
        cfg.depth_min = g->depth_min;
        cfg.depth_max = g->depth_max;
        cfg.max_width = g->max_width;
        cfg.avg_load = rat(g->avg_load_num, g->avg_load_den);
        cfg.load_jitter = g->load_jitter;
        cfg.edge_density = g->edge_density;
        cfg.seed = g->seed;
        cfg.integer_loads = g->integer_loads != 0;
        cfg.exact_mean = g->exact_mean != 0;
        cfg.t_min = rat(g->tmin_num, g->tmin_den);
        // the reference's own Theorem-1 check (experiment.cpp:163-240)
        ValidationSummary s = run_validation(cfg, corpus_size, platform_of(p), samples, rat(smin_num, smin_den),
                                             rat(smax_num, smax_den), parallel != 0);
        out[0] = s.tasks;
        out[1] = s.runs;
        out[2] = s.violations;
        dbl[0] = s.mean_tightness_worst;
        dbl[1] = s.mean_tightness_scaled;
    });
}

extern "C" char* ref_run_experiment(char sweep, const long long* values, int n_values, const ds_gen_config* g,
                                    const ds_platform* p, int corpus_size, uint32_t methods, int normalize_to) {
    std::string text;
    int st = guarded([&] {
        ExperimentSpec spec;
        spec.sweep = sweep == 'M' ? ExperimentSpec::SweepVar::sm_count
                     : sweep == 'P' ? ExperimentSpec::SweepVar::max_width
                                    : ExperimentSpec::SweepVar::depth;
        spec.values.assign(values, values + n_values);
        spec.base.depth_min = g->depth_min;
        spec.base.depth_max = g->depth_max;
        spec.base.max_width = g->max_width;
        spec.base.avg_load = rat(g->avg_load_num, g->avg_load_den);
        spec.base.load_jitter = g->load_jitter;
        spec.base.edge_density = g->edge_density;
        spec.base.seed = g->seed;
        spec.base.integer_loads = g->integer_loads != 0;
        spec.base.exact_mean = g->exact_mean != 0;
        spec.base.t_min = rat(g->tmin_num, g->tmin_den);
        spec.platform = platform_of(p);
        spec.corpus_size = corpus_size;
        const Method all[4] = {Method::proposed, Method::greedy, Method::greedy_unaware, Method::graham_para};
        spec.methods.clear();
        for (int k = 0; k < 4; ++k)
            if (methods & (1u << k)) spec.methods.push_back(all[k]);
        spec.normalize_to = all[normalize_to];
        // the reference's own sweep driver and CSV writer (experiment.cpp:81-161)
        std::ostringstream out;
        write_csv(run_experiment(spec), out);
        text = out.str();
    });
    return st == DS_OK ? dup(text) : nullptr;
}

// ---------------------------------------------------------------------------
// Simulator, task I/O and run_benchmarks (simulator.cpp, task_io.cpp,
// experiment.cpp:242-307), through the reference's own functions.
#include "dagsched/simulator.hpp"

#include <fstream>

namespace {
TimeModel time_model(int scaled, uint64_t seed, int64_t smin_n, int64_t smin_d, int64_t smax_n, int64_t smax_d) {
    TimeModel t;
    t.kind = scaled ? TimeModel::Kind::scaled : TimeModel::Kind::worst_case;
    t.seed = seed;
    if (scaled) {
        t.scale_min = rat(smin_n, smin_d);
        t.scale_max = rat(smax_n, smax_d);
    }
    return t;
}
}  // namespace

extern "C" int ref_sim_greedy(void* h, const ds_platform* p, int policy, uint64_t policy_seed, int runs, int scaled,
                              uint64_t time_seed, int64_t smin_n, int64_t smin_d, int64_t smax_n, int64_t smax_d,
                              int32_t* status, int64_t* makespan) {
    auto* c = static_cast<Corpus*>(h);
    for (uint64_t d = 0; d < c->n_dags; ++d) {
        for (int r = 0; r < runs; ++r) {
            status[d * runs + r] = DS_EINVAL;
            makespan[2 * (d * runs + r)] = makespan[2 * (d * runs + r) + 1] = 0;
        }
    }
    for (std::size_t i = 0; i < c->tasks.size(); ++i) {
        const uint64_t d = c->index[i];
        for (int r = 0; r < runs; ++r) {
            SimTrace tr;
            int st = guarded([&] {
                SimConfig cfg;
                cfg.platform = platform_of(p);
                cfg.mode = SimMode::greedy;
                cfg.policy = policy ? DispatchPolicy::random : DispatchPolicy::fifo;
                cfg.policy_seed = policy_seed + uint64_t(r);
                cfg.time_model = time_model(scaled, time_seed, smin_n, smin_d, smax_n, smax_d);
                tr = simulate_greedy(c->tasks[i], cfg);
            });
            if (st == DS_OK && !put(tr.makespan, makespan + 2 * (d * runs + r))) st = DS_EOVERFLOW;
            status[d * runs + r] = st;
        }
    }
    return DS_OK;
}

extern "C" char* ref_sim_greedy_trace(void* h, uint64_t d, const ds_platform* p, int policy, uint64_t policy_seed,
                                      int scaled, uint64_t time_seed, int64_t smin_n, int64_t smin_d, int64_t smax_n,
                                      int64_t smax_d) {
    auto* c = static_cast<Corpus*>(h);
    std::string text;
    int st = guarded([&] {
        SimConfig cfg;
        cfg.platform = platform_of(p);
        cfg.mode = SimMode::greedy;
        cfg.policy = policy ? DispatchPolicy::random : DispatchPolicy::fifo;
        cfg.policy_seed = policy_seed;
        cfg.time_model = time_model(scaled, time_seed, smin_n, smin_d, smax_n, smax_d);
        std::ostringstream out;
        write_trace(simulate_greedy(c->tasks.at(d), cfg), out);
        text = out.str();
    });
    return st == DS_OK ? dup(text) : nullptr;
}

extern "C" char* ref_sim_scheme_trace(void* h, uint64_t d, const ds_platform* p, int scaled, uint64_t time_seed,
                                      int64_t smin_n, int64_t smin_d, int64_t smax_n, int64_t smax_d) {
    auto* c = static_cast<Corpus*>(h);
    std::string text;
    int st = guarded([&] {
        SimConfig cfg;
        cfg.platform = platform_of(p);
        cfg.mode = SimMode::scheme;
        cfg.time_model = time_model(scaled, time_seed, smin_n, smin_d, smax_n, smax_d);
        const DagTask& t = c->tasks.at(d);
        const ScheduleScheme sch = schedule(t, cfg.platform);
        SimTrace tr = simulate_scheme(t, sch, cfg);
        check_precedence(tr, sch);
        std::ostringstream out;
        write_trace(tr, out);
        text = out.str();
    });
    return st == DS_OK ? dup(text) : nullptr;
}

// read_task + write_task round trip; *status gets the DS code of read_task's failure
extern "C" char* ref_task_roundtrip(const char* json, int64_t min_n, int64_t min_d, int has_seed, uint64_t seed,
                                    int32_t* status) {
    std::string text;
    int st = guarded([&] {
        std::istringstream in(json);
        DagTask t = read_task(in, rat(min_n, min_d));
        std::ostringstream out;
        if (has_seed) write_task(t, out, seed);
        else write_task(t, out);
        text = out.str();
    });
    if (status) *status = st;
    return st == DS_OK ? dup(text) : nullptr;
}

extern "C" char* ref_run_benchmarks(const char* const* paths, int n_paths, const int* sms, int n_sms,
                                    const long long* avgs, int n_avgs, int greedy_runs, uint64_t seed) {
    std::string text;
    int st = guarded([&] {
        std::vector<std::string> ps(paths, paths + n_paths);
        std::vector<int> ms(sms, sms + n_sms);
        std::vector<long long> as(avgs, avgs + n_avgs);
        std::ostringstream out;
        write_bench_table(run_benchmarks(ps, ms, as, greedy_runs, seed), out);
        text = out.str();
    });
    return st == DS_OK ? dup(text) : nullptr;
}

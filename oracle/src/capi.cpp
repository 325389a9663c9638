// TEST INFRASTRUCTURE — C wrapper (prefix orc_) over the oracle restatement,
// same contract as oracle/ref_capi.cpp (see oracle/oracle_api.h).
#include "oracle_api.h"
#include "restate.hpp"

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>

using namespace orc;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return DS_OK;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return DS_EOVERFLOW;
    } catch (const std::invalid_argument& e) {
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
    std::vector<Dag> dags;
    std::vector<uint64_t> index;
    uint64_t n_dags = 0;
};

Platform plat_of(const ds_platform* p) {
    Platform pl;
    pl.M = p->sm_count;
    pl.tmin = Q::of(p->tmin_num, p->tmin_den);
    return pl;
}

bool put(const Q& q, int64_t* slot) {
    if (q.n > INT64_MAX || q.n < INT64_MIN || q.d > INT64_MAX) return false;
    slot[0] = int64_t(q.n);
    slot[1] = int64_t(q.d);
    return true;
}

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_free(void* p) { std::free(p); }

void* orc_corpus_from_packed(const ds_dag_batch* b, int64_t mn, int64_t md, int32_t* status) {
    auto c = std::make_unique<Corpus>();
    c->n_dags = b->n_dags;
    for (uint64_t d = 0; d < b->n_dags; ++d) {
        std::vector<Q> loads;
        std::vector<std::pair<long long, long long>> edges;
        for (uint32_t i = b->node_off[d]; i < b->node_off[d + 1]; ++i) {
            loads.push_back(Q::of(b->load_num[i - b->node_off[0]], b->load_den ? b->load_den[i - b->node_off[0]] : 1));
        }
        for (uint32_t e = b->edge_off[d]; e < b->edge_off[d + 1]; ++e) {
            edges.emplace_back(b->edges[e - b->edge_off[0]] >> 16, b->edges[e - b->edge_off[0]] & 0xffffu);
        }
        int st = guarded([&] {
            c->dags.push_back(make_dag(std::move(loads), std::move(edges), Q::of(mn, md)));
            c->index.push_back(d);
        });
        if (status) status[d] = st;
    }
    return c.release();
}

void* orc_corpus_generate(const ds_gen_config* g, int64_t count) {
    auto c = std::make_unique<Corpus>();
    GenCfg cfg;
    cfg.depth_min = g->depth_min;
    cfg.depth_max = g->depth_max;
    cfg.max_width = g->max_width;
    cfg.avg_load = Q::of(g->avg_load_num, g->avg_load_den);
    cfg.jitter = g->load_jitter;
    cfg.density = g->edge_density;
    cfg.integer_loads = g->integer_loads != 0;
    cfg.exact_mean = g->exact_mean != 0;
    cfg.tmin = Q::of(g->tmin_num, g->tmin_den);
    if (count < 1) {
        g_err = "count must be >= 1";
        return nullptr;
    }
    c->dags.resize(count);
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : bad)
    for (int64_t i = 0; i < count; ++i) {
        GenCfg ci = cfg;
        ci.seed = g->seed + uint64_t(i);  // generator.cpp:102-106
        bad += guarded([&] { c->dags[i] = generate(ci); }) != DS_OK;
    }
    if (bad) return nullptr;
    c->n_dags = count;
    for (int64_t i = 0; i < count; ++i) c->index.push_back(uint64_t(i));
    return c.release();
}

int orc_corpus_size(void* h, uint64_t* n_dags, uint64_t* n_nodes, uint64_t* n_edges) {
    auto* c = static_cast<Corpus*>(h);
    uint64_t nn = 0, ne = 0;
    for (const Dag& g : c->dags) {
        nn += g.n;
        ne += g.edges.size();
    }
    *n_dags = c->dags.size();
    *n_nodes = nn;
    *n_edges = ne;
    return DS_OK;
}

int orc_corpus_pack(void* h, uint32_t* node_off, uint32_t* edge_off, int64_t* load_num,
                    int64_t* load_den, uint32_t* edges) {
    auto* c = static_cast<Corpus*>(h);
    uint32_t no = 0, eo = 0;
    for (size_t d = 0; d < c->dags.size(); ++d) {
        const Dag& g = c->dags[d];
        node_off[d] = no;
        edge_off[d] = eo;
        for (int i = 0; i < g.n; ++i) {
            int64_t s[2];
            if (!put(g.load[i], s)) return DS_EOVERFLOW;
            load_num[no] = s[0];
            load_den[no] = s[1];
            ++no;
        }
        for (auto [u, v] : g.edges) edges[eo++] = (uint32_t(u) << 16) | uint32_t(v);
    }
    node_off[c->dags.size()] = no;
    edge_off[c->dags.size()] = eo;
    return DS_OK;
}

void orc_corpus_free(void* h) { delete static_cast<Corpus*>(h); }

double orc_corpus_evaluate(void* h, const ds_platform* p, uint32_t mask, int parallel,
                           int32_t* status, int64_t* bounds) {
    auto* c = static_cast<Corpus*>(h);
    const Platform pl = plat_of(p);
    const long long n = (long long)c->dags.size();
    auto one = [&](long long i) {
        const Dag& g = c->dags[i];
        uint64_t d = c->index[i];
        int64_t* b = bounds + d * 10;
        Q v[5];
        // experiment.cpp:27-39 in method order, then lower_bound
        int st = guarded([&] {
            if (mask & DS_M_PROPOSED) v[0] = proposed_bound(schedule(g, pl));
            if (mask & DS_M_GREEDY) v[1] = greedy_bound(g, pl);
            if (mask & DS_M_GREEDY_UNAWARE) v[2] = greedy_unaware_bound(g, pl);
            if (mask & DS_M_GRAHAM_PARA) v[3] = graham_para_bound(g, pl);
            if (mask & DS_M_LOWER) v[4] = lower_bound(g, pl);
        });
        for (int k = 0; k < 10; ++k) b[k] = 0;
        if (st == DS_OK) {
            for (int k = 0; k < 5; ++k) {
                if ((mask >> k) & 1) {
                    if (!put(v[k], b + 2 * k)) st = DS_EOVERFLOW;
                }
            }
        }
        if (st != DS_OK) for (int k = 0; k < 10; ++k) b[k] = 0;  // failed DAGs carry no bounds
        if (status) status[d] = st;
    };
    auto t0 = std::chrono::steady_clock::now();
    if (parallel) {
#pragma omp parallel for schedule(dynamic)
        for (long long i = 0; i < n; ++i) one(i);
    } else {
        for (long long i = 0; i < n; ++i) one(i);
    }
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
}

char* orc_scheme_json(void* h, uint64_t d, const ds_platform* p) {
    auto* c = static_cast<Corpus*>(h);
    std::string text;
    int st = guarded([&] { text = scheme_json(schedule(c->dags.at(d), plat_of(p))); });
    return st == DS_OK ? dup(text) : nullptr;
}

char* orc_analyze_json(void* h, uint64_t d, const ds_platform* p) {
    auto* c = static_cast<Corpus*>(h);
    std::string text;
    int st = guarded([&] {
        const Dag& g = c->dags.at(d);
        const Platform pl = plat_of(p);
        Scheme s = schedule(g, pl);
        Q prop = proposed_bound(s), gr = greedy_bound(g, pl), gu = greedy_unaware_bound(g, pl),
          gp = graham_para_bound(g, pl), lo = lower_bound(g, pl);
        std::ostringstream o;
        o << "{\"per_group_response\": [";
        for (size_t i = 0; i < s.groups.size(); ++i) {
            o << (i ? ", " : "") << '"' << q_str(s.groups[i].resp) << '"';
        }
        // analysis.cpp:94-97: ratios against greedy_unaware
        o << "], \"proposed\": \"" << q_str(prop) << "\", \"greedy\": \"" << q_str(gr)
          << "\", \"greedy_unaware\": \"" << q_str(gu) << "\", \"graham_para\": \"" << q_str(gp)
          << "\", \"lower\": \"" << q_str(lo) << "\", \"normalized\": {\"graham_para\": \""
          << q_str(gp / gu) << "\", \"greedy\": \"" << q_str(gr / gu)
          << "\", \"greedy_unaware\": \"1\", \"proposed\": \"" << q_str(prop / gu) << "\"}}";
        text = o.str();
    });
    return st == DS_OK ? dup(text) : nullptr;
}

}  // extern "C"

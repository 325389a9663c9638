// Host corpus generation — replaces generate_corpus (generator.cpp:98-108).
//
// Stays on the CPU so every DAG is bit-identical to the reference's (the
// RNG call order of generator.cpp:24-96 is the contract: depth; widths; per
// node in layer order the parent draw then one coin per earlier-layer node
// except the parent; loads in id order; llround to the t_min grid; clamp).
// Emits the packed batch directly (no per-DAG objects), in parallel over
// seeds, into pageable or pinned arrays owned by a handle.
#include "../../include/dagsched_b200.h"

#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace ds {
int fail(int code, const std::string& msg);
}
#include "k5_generate_host.h"

namespace {

using i128 = __int128;

i128 gcd128(i128 a, i128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        i128 t = a % b;
        a = b;
        b = t;
    }
    return a;
}

struct Frac {  // exact non-negative rational for exact_mean rescaling
    i128 n = 0, d = 1;
    static Frac make(i128 n, i128 d) {
        i128 g = gcd128(n, d);
        if (g > 1) {
            n /= g;
            d /= g;
        }
        return Frac{n, d};
    }
};
Frac operator+(Frac a, Frac b) { return Frac::make(a.n * b.d + b.n * a.d, a.d * b.d); }
Frac operator*(Frac a, Frac b) { return Frac::make(a.n * b.n, a.d * b.d); }
bool operator<(Frac a, Frac b) { return a.n * b.d < b.n * a.d; }

struct Cfg {
    int dmin, dmax, width;
    double jitter, density, avg_d, tmin_d;
    bool integer_loads, exact_mean;
    Frac avg, tmin;
};

struct Dag {
    std::vector<Frac> loads;
    std::vector<uint32_t> edges;  // (u << 16) | v, sorted
};

void generate_one(const Cfg& c, uint64_t seed, Dag& out) {
    std::mt19937_64 rng(seed);
    const int depth = std::uniform_int_distribution<int>(c.dmin, c.dmax)(rng);
    int begin[512], size[512];
    int L = 0, next = 0;
    begin[L] = next;
    size[L++] = 1;
    next = 1;
    for (int l = 0; l < depth - 2; ++l) {
        const int w = std::uniform_int_distribution<int>(2, c.width)(rng);
        begin[L] = next;
        size[L++] = w;
        next += w;
    }
    const int sink = next++;
    out.edges.clear();
    std::vector<char> has_child(next, 0);
    std::uniform_real_distribution<double> coin(0.0, 1.0);
    for (int l = 1; l < L; ++l) {
        for (int v = begin[l]; v < begin[l] + size[l]; ++v) {
            const int parent =
                begin[l - 1] + int(std::uniform_int_distribution<std::size_t>(0, size[l - 1] - 1)(rng));
            out.edges.push_back(uint32_t(parent) << 16 | uint32_t(v));
            has_child[parent] = 1;
            for (int e = 0; e < l; ++e) {
                for (int u = begin[e]; u < begin[e] + size[e]; ++u) {
                    if (u != parent && coin(rng) < c.density) {
                        out.edges.push_back(uint32_t(u) << 16 | uint32_t(v));
                        has_child[u] = 1;
                    }
                }
            }
        }
    }
    for (int v = 0; v < sink; ++v) {
        if (!has_child[v]) out.edges.push_back(uint32_t(v) << 16 | uint32_t(sink));
    }
    std::sort(out.edges.begin(), out.edges.end());  // DagTask::make sorts (dag.cpp:49)
    std::uniform_real_distribution<double> ld(c.avg_d * (1.0 - c.jitter), c.avg_d * (1.0 + c.jitter));
    out.loads.resize(next);
    for (int v = 0; v < next; ++v) {
        const double x = ld(rng);
        Frac l = c.integer_loads ? Frac::make(i128(std::llround(x / c.tmin_d)), 1) * c.tmin
                                 : Frac::make(i128(std::llround(x * 1000.0)), 1000);
        if (l < c.tmin) l = c.tmin;
        out.loads[v] = l;
    }
    if (c.exact_mean) {
        Frac sum;
        for (const Frac& l : out.loads) sum = sum + l;
        const Frac f = Frac::make(c.avg.n * i128(next) * sum.d, c.avg.d * sum.n);
        for (Frac& l : out.loads) {
            l = l * f;
            if (l < c.tmin) l = c.tmin;
        }
    }
}

struct Corpus {
    bool pinned = false;
    float gen_ms = 0.f;  // device generation (DS_F_GPU_GENERATE): kernels + scans
    uint64_t n = 0, nn = 0, ne = 0;
    uint32_t *node_off = nullptr, *edge_off = nullptr, *edges = nullptr;
    int64_t *load_num = nullptr, *load_den = nullptr;
};

void* host_alloc(size_t bytes, bool pinned) {
    bytes = std::max<size_t>(bytes, 8);
    if (pinned) {
        void* p = nullptr;
        if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) return nullptr;
        return p;
    }
    return std::malloc(bytes);
}
void host_free(void* p, bool pinned) {
    if (!p) return;
    if (pinned) cudaFreeHost(p);
    else std::free(p);
}

void corpus_free(Corpus* c) {
    if (!c) return;
    host_free(c->node_off, c->pinned);
    host_free(c->edge_off, c->pinned);
    host_free(c->edges, c->pinned);
    host_free(c->load_num, c->pinned);
    host_free(c->load_den, c->pinned);
    delete c;
}

}  // namespace

extern "C" {

int ds_corpus_generate(const ds_gen_config* g, int64_t count, uint32_t flags, void** handle) {
    using ds::fail;
    if (!g || !handle) return fail(DS_EINVAL, "NULL argument");
    *handle = nullptr;
    // generator.cpp:9-22 (GenConfig::check) and :98-100
    if (count < 1) return fail(DS_EINVAL, "count must be >= 1");
    if (g->depth_min < 2 || g->depth_max < g->depth_min)
        return fail(DS_EINVAL, "depth range must satisfy 2 <= min <= max");
    if (g->max_width < 2) return fail(DS_EINVAL, "max_width must be >= 2");
    if (g->tmin_den <= 0 || g->tmin_num <= 0) return fail(DS_EINVAL, "t_min must be positive");
    if (g->avg_load_den <= 0) return fail(DS_EINVAL, "avg_load denominator must be positive");
    if (g->load_jitter < 0 || g->load_jitter > 1) return fail(DS_EINVAL, "load_jitter must be in [0, 1]");
    if (g->edge_density < 0 || g->edge_density > 1) return fail(DS_EINVAL, "edge_density must be in [0, 1]");
    Cfg c;
    c.dmin = g->depth_min;
    c.dmax = g->depth_max;
    c.width = g->max_width;
    c.jitter = g->load_jitter;
    c.density = g->edge_density;
    c.integer_loads = g->integer_loads != 0;
    c.exact_mean = g->exact_mean != 0;
    c.avg = Frac::make(g->avg_load_num, g->avg_load_den);
    c.tmin = Frac::make(g->tmin_num, g->tmin_den);
    if (c.avg < c.tmin) return fail(DS_EINVAL, "avg_load must be >= t_min");
    c.avg_d = double(g->avg_load_num) / double(g->avg_load_den);
    c.tmin_d = double(g->tmin_num) / double(g->tmin_den);
    // the packed form indexes nodes in 16 bits and generate_one keeps <= 512
    // layers; a generated DAG above DS_MAX_NODES gets DS_ETOOBIG from the
    // analysis, like any other
    if (c.dmax > 513 || 2 + int64_t(c.dmax - 2) * c.width > 65535)
        return fail(DS_ETOOBIG, "generated DAGs could exceed 65535 nodes or 512 layers");
    if (flags & DS_F_GPU_GENERATE) {
        if (2 + int64_t(c.dmax - 2) * c.width > 256)
            return fail(DS_ETOOBIG, "GPU generation (K5) covers DAGs up to 256 nodes; generate larger ones on the host");
        ds::K5Params p;
        p.count = uint64_t(count);
        p.seed = g->seed;
        p.dmin = c.dmin;
        p.dmax = c.dmax;
        p.width = c.width;
        p.integer_loads = c.integer_loads;
        p.exact_mean = c.exact_mean;
        p.lo = c.avg_d * (1.0 - c.jitter);  // the load distribution's bounds (generator.cpp:62-63)
        p.hi = c.avg_d * (1.0 + c.jitter);
        p.tmin_f = c.tmin_d;
        p.density = c.density;
        p.tmin_n = uint64_t(c.tmin.n);
        p.tmin_d = uint64_t(c.tmin.d);
        p.avg_n = uint64_t(c.avg.n);
        p.avg_d = uint64_t(c.avg.d);
        auto* cp = new Corpus();
        cp->pinned = flags & DS_F_PINNED;
        cp->n = uint64_t(count);
        int device = 0;
        if (cudaGetDevice(&device) != cudaSuccess) device = 0;
        auto alloc = [](uint64_t nn, uint64_t ne, void* user, ds::K5Host* h) -> int {
            auto* cp = static_cast<Corpus*>(user);
            cp->nn = nn;
            cp->ne = ne;
            cp->node_off = static_cast<uint32_t*>(host_alloc((cp->n + 1) * 4, cp->pinned));
            cp->edge_off = static_cast<uint32_t*>(host_alloc((cp->n + 1) * 4, cp->pinned));
            cp->edges = static_cast<uint32_t*>(host_alloc(ne * 4, cp->pinned));
            cp->load_num = static_cast<int64_t*>(host_alloc(nn * 8, cp->pinned));
            cp->load_den = static_cast<int64_t*>(host_alloc(nn * 8, cp->pinned));
            if (!cp->node_off || !cp->edge_off || !cp->edges || !cp->load_num || !cp->load_den)
                return ds::fail(DS_ENOMEM, "host allocation failed");
            *h = ds::K5Host{cp->node_off, cp->edge_off, cp->edges, cp->load_num, cp->load_den};
            return DS_OK;
        };
        const int words = 2 + int64_t(c.dmax - 2) * c.width <= 64 ? 1 : 4;
        const int rc = ds::k5_generate_host(p, words, device, alloc, cp, &cp->gen_ms);
        if (rc != DS_OK) {
            corpus_free(cp);
            return rc;
        }
        *handle = cp;
        return DS_OK;
    }

    // pass 1: generate in parallel into per-thread buffers (chunked by seed)
    const int nt = std::max(1, omp_get_max_threads());
    const int64_t per = (count + nt - 1) / nt;
    std::vector<std::vector<uint32_t>> t_nodes(nt), t_edges(nt), t_ecount(nt);
    std::vector<std::vector<int64_t>> t_num(nt), t_den(nt);
    int bad = 0;
#pragma omp parallel num_threads(nt) reduction(+ : bad)
    {
        const int t = omp_get_thread_num();
        const int64_t lo = std::min<int64_t>(count, per * t), hi = std::min<int64_t>(count, lo + per);
        Dag dag;
        auto& tn = t_nodes[t];
        auto& te = t_edges[t];
        auto& tc = t_ecount[t];
        auto& nu = t_num[t];
        auto& de = t_den[t];
        for (int64_t i = lo; i < hi; ++i) {
            generate_one(c, g->seed + uint64_t(i), dag);
            tn.push_back(uint32_t(dag.loads.size()));
            tc.push_back(uint32_t(dag.edges.size()));
            te.insert(te.end(), dag.edges.begin(), dag.edges.end());
            for (const Frac& l : dag.loads) {
                if (l.n > INT64_MAX || l.d > INT64_MAX) ++bad;
                nu.push_back(int64_t(l.n));
                de.push_back(int64_t(l.d));
            }
        }
    }
    if (bad) return fail(DS_EOVERFLOW, "generated load outside int64");
    auto* cp = new Corpus();
    cp->pinned = flags & DS_F_PINNED;
    cp->n = uint64_t(count);
    for (int t = 0; t < nt; ++t) {
        cp->nn += t_num[t].size();
        cp->ne += t_edges[t].size();
    }
    if (cp->nn > 0xffffffffull || cp->ne > 0xffffffffull) {
        corpus_free(cp);
        return fail(DS_ETOOBIG, "batch exceeds 2^32 nodes or edges");
    }
    cp->node_off = static_cast<uint32_t*>(host_alloc((cp->n + 1) * 4, cp->pinned));
    cp->edge_off = static_cast<uint32_t*>(host_alloc((cp->n + 1) * 4, cp->pinned));
    cp->edges = static_cast<uint32_t*>(host_alloc(cp->ne * 4, cp->pinned));
    cp->load_num = static_cast<int64_t*>(host_alloc(cp->nn * 8, cp->pinned));
    cp->load_den = static_cast<int64_t*>(host_alloc(cp->nn * 8, cp->pinned));
    if (!cp->node_off || !cp->edge_off || !cp->edges || !cp->load_num || !cp->load_den) {
        corpus_free(cp);
        return fail(DS_ENOMEM, "host allocation failed");
    }
    // pass 2: prefix offsets per thread, then parallel copy-out
    std::vector<uint64_t> dag0(nt + 1, 0), node0(nt + 1, 0), edge0(nt + 1, 0);
    for (int t = 0; t < nt; ++t) {
        dag0[t + 1] = dag0[t] + t_nodes[t].size();
        node0[t + 1] = node0[t] + t_num[t].size();
        edge0[t + 1] = edge0[t] + t_edges[t].size();
    }
#pragma omp parallel for num_threads(nt) schedule(static, 1)
    for (int t = 0; t < nt; ++t) {
        uint64_t d = dag0[t], no = node0[t], eo = edge0[t];
        for (size_t k = 0; k < t_nodes[t].size(); ++k, ++d) {
            cp->node_off[d] = uint32_t(no);
            cp->edge_off[d] = uint32_t(eo);
            no += t_nodes[t][k];
            eo += t_ecount[t][k];
        }
        if (!t_num[t].empty()) {
            std::memcpy(cp->load_num + node0[t], t_num[t].data(), t_num[t].size() * 8);
            std::memcpy(cp->load_den + node0[t], t_den[t].data(), t_den[t].size() * 8);
        }
        if (!t_edges[t].empty()) std::memcpy(cp->edges + edge0[t], t_edges[t].data(), t_edges[t].size() * 4);
    }
    cp->node_off[cp->n] = uint32_t(cp->nn);
    cp->edge_off[cp->n] = uint32_t(cp->ne);
    *handle = cp;
    return DS_OK;
}

int ds_corpus_view(void* handle, ds_dag_batch* view) {
    auto* c = static_cast<Corpus*>(handle);
    if (!c || !view) return ds::fail(DS_EINVAL, "NULL argument");
    view->n_dags = c->n;
    view->node_off = c->node_off;
    view->edge_off = c->edge_off;
    view->load_num = c->load_num;
    view->load_den = c->load_den;
    view->edges = c->edges;
    return DS_OK;
}

float ds_corpus_gen_ms(void* handle) {
    auto* c = static_cast<Corpus*>(handle);
    return c ? c->gen_ms : 0.f;
}

void ds_corpus_free(void* handle) { corpus_free(static_cast<Corpus*>(handle)); }

}  // extern "C"

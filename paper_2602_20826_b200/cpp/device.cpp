// Kept C++ API — packing and status mapping over the C-ABI.
#include "device.hpp"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <thread>

namespace dagsched::detail {

void parallel_for(std::size_t n, const std::function<void(std::size_t, std::size_t)>& f, std::size_t min_chunk) {
    const std::size_t hw = std::max(1u, std::thread::hardware_concurrency());
    const std::size_t parts = std::max<std::size_t>(1, std::min(hw, n / std::max<std::size_t>(1, min_chunk)));
    if (parts <= 1) {
        f(0, n);
        return;
    }
    std::vector<std::exception_ptr> err(parts);
    std::vector<std::thread> th;
    for (std::size_t i = 0; i < parts; ++i) {
        th.emplace_back([&, i] {
            try {
                f(n * i / parts, n * (i + 1) / parts);
            } catch (...) {
                err[i] = std::current_exception();
            }
        });
    }
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

struct Packed::Store {
    std::unique_lock<std::mutex> lease;      // the pinned arena, held while the batch lives
    std::unique_ptr<unsigned char[]> heap;   // else a heap block (default-initialised: untouched)
};

namespace {
struct PinnedArena {
    std::mutex mu;
    void* p = nullptr;
    std::size_t cap = 0;
};
PinnedArena& pinned_arena() {
    static PinnedArena* a = new PinnedArena;  // never destroyed: cudaFreeHost after the runtime's teardown is unsafe
    return *a;
}
bool arena_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DAGSCHED_PINNED_ARENA");
        return !(e && e[0] == '0');
    }();
    return on;
}
constexpr std::size_t kArenaMin = std::size_t(4) << 20;  // smaller batches: heap (the latency path copies anyway)

// `bytes` of storage for a batch: the arena when it is free and big enough
// (grown on demand), else the heap
unsigned char* acquire(Packed& p, std::size_t bytes) {
    p.store = std::make_shared<Packed::Store>();
    if (bytes >= kArenaMin && arena_enabled()) {
        PinnedArena& a = pinned_arena();
        std::unique_lock<std::mutex> lk(a.mu, std::try_to_lock);
        if (lk.owns_lock()) {
            if (a.cap < bytes) {
                if (a.p) ds_pinned_free(a.p);
                a.p = nullptr;
                a.cap = 0;
                const std::size_t want = bytes + bytes / 4;
                if (ds_pinned_alloc(want, &a.p) == DS_OK) a.cap = want;
            }
            if (a.cap >= bytes) {
                p.store->lease = std::move(lk);
                p.pinned = true;
                return static_cast<unsigned char*>(a.p);
            }
        }
    }
    p.store->heap.reset(new unsigned char[bytes ? bytes : 1]);
    return p.store->heap.get();
}
}  // namespace

Packed pack(const std::vector<const DagTask*>& tasks, bool with_results) {
    Packed p;
    const std::size_t nd = tasks.size();
    p.n_dags = nd;
    // the host's cores each take a contiguous run of tasks, the same runs in
    // every pass below
    const std::size_t hw = std::max(1u, std::thread::hardware_concurrency());
    const std::size_t parts = std::max<std::size_t>(1, std::min(hw, nd / 2048));
    auto run = [&](std::size_t i) { return nd * i / parts; };
    std::vector<std::size_t> pn(parts + 1, 0), pe(parts + 1, 0);
    parallel_for(parts, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            std::size_t a = 0, b = 0;
            for (std::size_t d = run(i); d < run(i + 1); ++d) {
                if (tasks[d]->size() > DS_MAX_NODES) throw std::invalid_argument("DAG larger than DS_MAX_NODES nodes");
                a += tasks[d]->size();
                b += tasks[d]->edges().size();
            }
            pn[i + 1] = a;
            pe[i + 1] = b;
        }
    }, 1);
    for (std::size_t i = 0; i < parts; ++i) {
        pn[i + 1] += pn[i];
        pe[i + 1] += pe[i];
    }
    p.n_nodes = pn[parts];
    p.n_edges = pe[parts];
    if (p.n_nodes > 0xffffffffull || p.n_edges > 0xffffffffull)
        throw std::invalid_argument("batch exceeds 2^32 nodes or edges");
    // layout (8-byte aligned): num, den, bounds | node_off, edge_off, edges, status
    const std::size_t N = p.n_nodes, E = p.n_edges, R = with_results ? nd : 0;
    const std::size_t bytes = 8 * (2 * N + 10 * R) + 4 * (2 * (nd + 1) + E + R) + 64;
    unsigned char* base = acquire(p, bytes);
    p.num = reinterpret_cast<std::int64_t*>(base);
    p.den = p.num + N;
    p.bounds = with_results ? p.den + N : nullptr;
    p.node_off = reinterpret_cast<std::uint32_t*>(p.den + N + 10 * R);
    p.edge_off = p.node_off + nd + 1;
    p.edges = p.edge_off + nd + 1;
    p.status = with_results ? reinterpret_cast<std::int32_t*>(p.edges + E) : nullptr;
    p.node_off[0] = 0;
    p.edge_off[0] = 0;
    std::atomic<bool> frac{false};
    constexpr BigInt::u128 kMax = BigInt::u128(INT64_MAX);
    parallel_for(parts, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t r = lo; r < hi; ++r) {
            bool f = false;
            std::size_t i = pn[r], e = pe[r];
            for (std::size_t d = run(r); d < run(r + 1); ++d) {
                const DagTask& t = *tasks[d];
                for (const DagNode& v : t.nodes()) {
                    const BigInt& n = v.load.num();
                    const BigInt& dn = v.load.den();
                    if (n.magnitude() > kMax || dn.magnitude() > kMax)
                        throw std::overflow_error("load outside the C-ABI's int64 range");
                    p.num[i++] = n.negative() ? -std::int64_t(n.magnitude()) : std::int64_t(n.magnitude());
                    f |= dn.magnitude() != 1;
                }
                t.edge_words_into(p.edges + e);
                e += t.edges().size();
                p.node_off[d + 1] = std::uint32_t(i);
                p.edge_off[d + 1] = std::uint32_t(e);
            }
            if (f) frac = true;
        }
    }, 1);
    p.integer = !frac;
    if (!p.integer) {  // denominators only when some load is fractional
        parallel_for(parts, [&](std::size_t lo, std::size_t hi) {
            for (std::size_t r = lo; r < hi; ++r) {
                std::size_t i = pn[r];
                for (std::size_t d = run(r); d < run(r + 1); ++d)
                    for (const DagNode& v : tasks[d]->nodes()) p.den[i++] = std::int64_t(v.load.den().magnitude());
            }
        }, 1);
    }
    return p;
}

Packed pack_compact(const std::vector<const DagTask*>& tasks, bool with_results) {
    const std::size_t nd = tasks.size();
    const std::size_t hw = std::max(1u, std::thread::hardware_concurrency());
    const std::size_t parts = std::max<std::size_t>(1, std::min(hw, nd / 2048));
    auto run = [&](std::size_t i) { return nd * i / parts; };
    // sizes: nodes and adjacency words per run; any DAG above 64 nodes -> wide form
    std::vector<std::size_t> pn(parts + 1, 0), pw(parts + 1, 0);
    std::atomic<bool> fits{nd > 0};
    parallel_for(parts, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            std::size_t a = 0, w = 0;
            for (std::size_t d = run(i); d < run(i + 1); ++d) {
                const std::size_t n = tasks[d]->size();
                if (n > 64) fits = false;
                a += n;
                w += (n * (n - 1) / 2 + 31) / 32;
            }
            pn[i + 1] = a;
            pw[i + 1] = w;
        }
    }, 1);
    if (!fits) return pack(tasks, with_results);
    for (std::size_t i = 0; i < parts; ++i) {
        pn[i + 1] += pn[i];
        pw[i + 1] += pw[i];
    }
    Packed p;
    p.n_dags = nd;
    p.n_nodes = pn[parts];
    p.tri = true;
    const std::size_t N = p.n_nodes, Wd = pw[parts], R = with_results ? nd : 0;
    if (N > 0xffffffffull || Wd > 0xffffffffull) return pack(tasks, with_results);
    // layout (8-byte aligned first): bounds | node_off, adj_off, adj, status | ln16
    const std::size_t bytes = 8 * 10 * R + 4 * (2 * (nd + 1) + Wd + R) + 2 * N + 64;
    unsigned char* base = acquire(p, bytes);
    p.bounds = with_results ? reinterpret_cast<std::int64_t*>(base) : nullptr;
    p.node_off = reinterpret_cast<std::uint32_t*>(base + 8 * 10 * R);
    p.adj_off = p.node_off + nd + 1;
    p.adj = p.adj_off + nd + 1;
    p.status = with_results ? reinterpret_cast<std::int32_t*>(p.adj + Wd) : nullptr;
    p.ln16 = reinterpret_cast<std::uint16_t*>(p.adj + Wd + R);
    p.node_off[0] = 0;
    p.adj_off[0] = 0;
    std::atomic<bool> ok{true};
    parallel_for(parts, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t r = lo; r < hi && ok; ++r) {
            std::size_t i = pn[r], w = pw[r];
            for (std::size_t d = run(r); d < run(r + 1); ++d) {
                const DagTask& t = *tasks[d];
                const std::size_t n = t.size();
                for (const DagNode& v : t.nodes()) {
                    const BigInt& num = v.load.num();
                    if (v.load.den().magnitude() != 1 || num.negative() || num.magnitude() > 0xffff) {
                        ok = false;
                        return;
                    }
                    p.ln16[i++] = std::uint16_t(num.magnitude());
                }
                const std::size_t nw = (n * (n - 1) / 2 + 31) / 32;
                std::fill(p.adj + w, p.adj + w + nw, 0u);
                if (!t.tri_bits_into(p.adj + w)) {
                    ok = false;
                    return;
                }
                w += nw;
                p.node_off[d + 1] = std::uint32_t(i);
                p.adj_off[d + 1] = std::uint32_t(w);
            }
        }
    }, 1);
    if (!ok) return pack(tasks, with_results);  // a fractional or >= 2^16 load, or a non-topological order
    return p;
}

ds_platform platform_of(const Platform& p) {
    p.check();
    return ds_platform{p.sm_count, DS_PF_PREMADE, to_int64(numerator(p.t_min)), to_int64(denominator(p.t_min))};
}

void raise(int st, const std::string& what) {
    switch (st) {
        case DS_OK: return;
        case DS_EINVAL: throw std::invalid_argument(what);
        case DS_EOVERFLOW: throw std::overflow_error(what);
        case DS_EINVARIANT: throw std::logic_error(what);
        case DS_E_LOAD: throw ValidationError(what + ": load below minimum");
        case DS_E_LOAD_TMIN: throw ValidationError(what + ": load below the platform time unit");
        default:
            if (st >= DS_E_EMPTY && st <= DS_E_LOAD_TMIN) throw ValidationError(what);
            throw std::runtime_error(what);
    }
}

void check(int rc) {
    if (rc != DS_OK) raise(rc, std::string("dagsched_b200: ") + ds_last_error());
}

std::vector<int> devices() {
    std::vector<int> out;
    if (const char* env = std::getenv("DAGSCHED_DEVICES")) {
        std::stringstream ss(env);
        std::string tok;
        while (std::getline(ss, tok, ',')) out.push_back(std::stoi(tok));
    }
    if (out.empty()) {
        int n = 0;
        check(ds_device_count(&n));
        for (int i = 0; i < n; ++i) out.push_back(i);
    }
    if (out.empty()) throw std::runtime_error("dagsched_b200: no CUDA device");
    return out;
}

}  // namespace dagsched::detail

// Kept C++ API — packing and status mapping over the C-ABI.
#include "device.hpp"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <exception>
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

Packed pack(const std::vector<const DagTask*>& tasks) {
    Packed p;
    const std::size_t nd = tasks.size();
    p.node_off.assign(nd + 1, 0);
    p.edge_off.assign(nd + 1, 0);
    for (std::size_t d = 0; d < nd; ++d) {
        if (tasks[d]->size() > DS_MAX_NODES) throw std::invalid_argument("DAG larger than DS_MAX_NODES nodes");
        p.node_off[d + 1] = p.node_off[d] + std::uint32_t(tasks[d]->size());
        p.edge_off[d + 1] = p.edge_off[d] + std::uint32_t(tasks[d]->edges().size());
    }
    p.num.resize(p.node_off[nd]);
    p.den.resize(p.node_off[nd]);
    p.edges.resize(p.edge_off[nd]);
    std::atomic<bool> frac{false};
    constexpr BigInt::u128 kMax = BigInt::u128(INT64_MAX);
    parallel_for(nd, [&](std::size_t lo, std::size_t hi) {
        bool f = false;
        for (std::size_t d = lo; d < hi; ++d) {
            std::size_t i = p.node_off[d];
            for (const DagNode& v : tasks[d]->nodes()) {
                const BigInt& n = v.load.num();
                const BigInt& dn = v.load.den();
                if (n.magnitude() > kMax || dn.magnitude() > kMax)
                    throw std::overflow_error("load outside the C-ABI's int64 range");
                p.num[i] = n.negative() ? -std::int64_t(n.magnitude()) : std::int64_t(n.magnitude());
                p.den[i] = std::int64_t(dn.magnitude());
                f |= p.den[i] != 1;
                ++i;
            }
            std::size_t e = p.edge_off[d];
            for (std::uint32_t w : tasks[d]->edge_words()) p.edges[e++] = w;
        }
        if (f) frac = true;
    });
    p.integer = !frac;
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

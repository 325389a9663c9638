// Kept C++ API — packing and status mapping over the C-ABI.
#include "device.hpp"

#include <cstdlib>
#include <sstream>
#include <stdexcept>

namespace dagsched::detail {

Packed pack(const std::vector<const DagTask*>& tasks) {
    Packed p;
    for (const DagTask* t : tasks) {
        for (const DagNode& v : t->nodes()) {
            if (numerator(v.load) > BigInt(INT64_MAX) || denominator(v.load) > BigInt(INT64_MAX))
                throw std::overflow_error("load outside the C-ABI's int64 range");
            p.num.push_back(to_int64(numerator(v.load)));
            p.den.push_back(to_int64(denominator(v.load)));
            p.integer &= p.den.back() == 1;
        }
        if (t->size() > DS_MAX_NODES) throw std::invalid_argument("DAG larger than DS_MAX_NODES nodes");
        for (std::uint32_t w : t->edge_words()) p.edges.push_back(w);
        p.node_off.push_back(std::uint32_t(p.num.size()));
        p.edge_off.push_back(std::uint32_t(p.edges.size()));
    }
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

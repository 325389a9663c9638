// Kept C++ API — generator: ds_corpus_generate (host, bit-identical to the
// reference's RNG call order) unpacked into DagTasks.
#include "dagsched/generator.hpp"

#include "device.hpp"

#include <algorithm>
#include <mutex>

namespace dagsched {

void GenConfig::check() const {
    if (depth_min < 2 || depth_max < depth_min) throw std::invalid_argument("depth range must satisfy 2 <= min <= max");
    if (max_width < 2) throw std::invalid_argument("max_width must be >= 2");
    if (t_min <= 0) throw std::invalid_argument("t_min must be positive");
    if (avg_load < t_min) throw std::invalid_argument("avg_load must be >= t_min");
    if (load_jitter < 0 || load_jitter > 1) throw std::invalid_argument("load_jitter must be in [0, 1]");
    if (edge_density < 0 || edge_density > 1) throw std::invalid_argument("edge_density must be in [0, 1]");
}

std::vector<DagTask> generate_corpus(const GenConfig& c, int count) {
    if (count < 1) throw std::invalid_argument("count must be >= 1");
    c.check();
    ds_gen_config g{c.depth_min, c.depth_max, c.max_width, c.integer_loads ? 1 : 0,
                    to_int64(numerator(c.avg_load)), to_int64(denominator(c.avg_load)), c.load_jitter,
                    c.edge_density, c.seed, to_int64(numerator(c.t_min)), to_int64(denominator(c.t_min)),
                    c.exact_mean ? 1 : 0, 0};
    void* h = nullptr;
    detail::check(ds_corpus_generate(&g, count, 0, &h));
    ds_dag_batch v;
    ds_corpus_view(h, &v);
    // DagTask::make per DAG on the host's cores (chunks kept in DAG order)
    std::mutex mu;
    std::vector<std::pair<std::size_t, std::vector<DagTask>>> done;
    try {
        detail::parallel_for(v.n_dags, [&](std::size_t lo, std::size_t hi) {
            std::vector<DagTask> mine;
            mine.reserve(hi - lo);
            for (std::size_t d = lo; d < hi; ++d) {
                std::vector<DagNode> nodes;
                std::vector<std::pair<NodeId, NodeId>> edges;
                nodes.reserve(v.node_off[d + 1] - v.node_off[d]);
                edges.reserve(v.edge_off[d + 1] - v.edge_off[d]);
                for (uint32_t i = v.node_off[d]; i < v.node_off[d + 1]; ++i)
                    nodes.push_back(
                        DagNode{i - v.node_off[d], Rational(BigInt(v.load_num[i]), BigInt(v.load_den[i]))});
                for (uint32_t e = v.edge_off[d]; e < v.edge_off[d + 1]; ++e)
                    edges.emplace_back(v.edges[e] >> 16, v.edges[e] & 0xffffu);
                mine.push_back(DagTask::make(std::move(nodes), std::move(edges), std::nullopt, c.t_min));
            }
            std::lock_guard<std::mutex> lock(mu);
            done.emplace_back(lo, std::move(mine));
        }, 1024);
    } catch (...) {
        ds_corpus_free(h);
        throw;
    }
    std::sort(done.begin(), done.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    std::vector<DagTask> out;
    out.reserve(count);
    for (auto& [lo, part] : done)
        for (DagTask& t : part) out.push_back(std::move(t));
    ds_corpus_free(h);
    return out;
}

DagTask generate(const GenConfig& config) { return std::move(generate_corpus(config, 1).front()); }

}  // namespace dagsched

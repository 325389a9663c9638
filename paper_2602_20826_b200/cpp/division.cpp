// Kept C++ API — division (Alg. 1). build_blocks/local_paths are host
// queries over the task's bitsets; build_groups is computed by the device
// (the K1 kernel's division phase via ds_schedule_batch).
#include "dagsched/division.hpp"

#include "device.hpp"

#include <algorithm>
#include <set>

namespace dagsched {

std::vector<Block> build_blocks(const DagTask& task) {
    std::vector<Block> out;
    std::set<NodeId> taken;
    for (NodeId j : task.join_nodes()) {
        Block b{j, {}};
        for (NodeId a : task.ancestors(j))
            if (taken.insert(a).second) b.members.push_back(a);
        out.push_back(std::move(b));
    }
    Block rest{std::nullopt, {}};
    for (const DagNode& v : task.nodes())
        if (!taken.count(v.id)) rest.members.push_back(v.id);
    out.push_back(std::move(rest));
    return out;
}

LocalPathSet local_paths(const DagTask& task, const Block& block) {
    const std::set<NodeId> in(block.members.begin(), block.members.end());
    LocalPathSet out;
    for (NodeId v : block.members) {
        const auto succ = task.successors(v);
        if (std::any_of(succ.begin(), succ.end(), [&](NodeId s) { return in.count(s) > 0; })) continue;
        std::vector<NodeId> rev{v};
        for (NodeId cur = v;;) {  // unique in-block predecessor chain
            std::optional<NodeId> up;
            for (NodeId p : task.predecessors(cur))
                if (in.count(p)) up = p;
            if (!up) break;
            rev.push_back(*up);
            cur = *up;
        }
        out.paths.emplace_back(rev.rbegin(), rev.rend());
    }
    return out;
}

BalancedGroupList build_groups(const DagTask& task, const Platform& platform) {
    const detail::Packed p = detail::pack({&task});
    const ds_dag_batch b = p.view();
    const ds_platform pl = detail::platform_of(platform);
    const std::size_t n = task.size();
    int32_t st = 0;
    uint16_t ne = 0, ng = 0, nd = 0;
    std::vector<int16_t> blk(n), div(n);
    ds_scheme_out out{&st, &ne, &ng, &nd, blk.data(), div.data(), nullptr, nullptr, nullptr, nullptr};
    detail::check(ds_schedule_batch(&b, &pl, &out, 0));
    // build_groups has no t_min check of its own (division.cpp:67-126): the
    // device still fills the division when only schedule() would refuse
    if (st != DS_E_LOAD_TMIN) detail::raise(st, "build_groups");
    BalancedGroupList g;
    g.groups.assign(nd, {});
    for (std::size_t i = 0; i < n; ++i) g.groups[div[i]].push_back(task.nodes()[i].id);
    return g;
}

}  // namespace dagsched

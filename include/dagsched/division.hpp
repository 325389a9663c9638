// dagsched_b200 — kept C++ API: sub-graph division (Alg. 1).
// Signatures of the reference's division.hpp:15-43. build_groups runs on the
// GPU (the K1 kernel's division phase, via ds_schedule_batch).
#pragma once

#include "dagsched/dag.hpp"
#include "dagsched/exec_model.hpp"

#include <optional>
#include <vector>

namespace dagsched {

struct Block {
    std::optional<NodeId> join;   // nullopt: the residual block
    std::vector<NodeId> members;  // id-sorted
};

struct LocalPathSet {
    std::vector<std::vector<NodeId>> paths;  // one per local sink, by sink id
};

struct BalancedGroupList {
    std::vector<std::vector<NodeId>> groups;  // the division Pi, each id-sorted
};

std::vector<Block> build_blocks(const DagTask& task);
LocalPathSet local_paths(const DagTask& task, const Block& block);
BalancedGroupList build_groups(const DagTask& task, const Platform& platform);

}  // namespace dagsched

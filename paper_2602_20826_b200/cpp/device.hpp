// Internal: the kept C++ API's bridge to the C-ABI (libdagsched_b200.so).
#pragma once

#include "../../include/dagsched_b200.h"
#include "dagsched/dag.hpp"
#include "dagsched/exec_model.hpp"

#include <string>
#include <vector>

namespace dagsched::detail {

struct Packed {
    std::vector<std::uint32_t> node_off{0}, edge_off{0}, edges;
    std::vector<std::int64_t> num, den;
    bool integer = true;
    ds_dag_batch view() const {
        return ds_dag_batch{node_off.size() - 1, node_off.data(), edge_off.data(), num.data(),
                            integer ? nullptr : den.data(), edges.data()};
    }
};

Packed pack(const std::vector<const DagTask*>& tasks);
ds_platform platform_of(const Platform& p);
// Throws the reference's exception type for a DS_* status.
void raise(int status, const std::string& what);
void check(int rc);
// Devices for batch work: $DAGSCHED_DEVICES (comma list) or every visible GPU.
std::vector<int> devices();

}  // namespace dagsched::detail

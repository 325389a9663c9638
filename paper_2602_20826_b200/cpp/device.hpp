// Internal: the kept C++ API's bridge to the C-ABI (libdagsched_b200.so).
#pragma once

#include "../../include/dagsched_b200.h"
#include "dagsched/dag.hpp"
#include "dagsched/exec_model.hpp"
#include "dagsched/scheduler.hpp"

#include <cstddef>
#include <functional>
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
// f(lo, hi) over [0, n) split into contiguous chunks on the host's cores
// (std::thread; the first exception, in chunk order, is rethrown). Host
// bookkeeping around the device calls: packing DagTasks, building results.
void parallel_for(std::size_t n, const std::function<void(std::size_t, std::size_t)>& f,
                  std::size_t min_chunk = 4096);
ds_platform platform_of(const Platform& p);
// Throws the reference's exception type for a DS_* status.
void raise(int status, const std::string& what);
void check(int rc);
// Devices for batch work: $DAGSCHED_DEVICES (comma list) or every visible GPU.
std::vector<int> devices();
// ds_schedule_batch over tasks (no copies) -> materialised schemes; with
// `bounds`, also the device's 5 bounds per task (num/den pairs, DS_BOUND_*).
std::vector<ScheduleScheme> schedule_ptrs(const std::vector<const DagTask*>& tasks, const Platform& platform,
                                          int device, std::vector<int64_t>* bounds);

}  // namespace dagsched::detail

// Internal: the kept C++ API's bridge to the C-ABI (libdagsched_b200.so).
#pragma once

#include "../../include/dagsched_b200.h"
#include "dagsched/dag.hpp"
#include "dagsched/exec_model.hpp"
#include "dagsched/scheduler.hpp"

#include <cstddef>
#include <functional>
#include <memory>
#include <string>
#include <vector>

namespace dagsched::detail {

// A batch of DagTasks in the C-ABI's packed form (ds_dag_batch), plus
// result staging (status[n_dags], bounds[10 n_dags]) when asked for. Large
// batches are packed into a process-wide pinned arena (the C-ABI's copies then
// run at full PCIe rate; one batch holds it at a time, others fall back to
// the heap; DAGSCHED_PINNED_ARENA=0 disables it); the arrays are filled by
// the host's cores, each first touching its own slice.
struct Packed {
    std::size_t n_dags = 0, n_nodes = 0, n_edges = 0;
    std::uint32_t *node_off = nullptr, *edge_off = nullptr, *edges = nullptr;
    std::int64_t *num = nullptr, *den = nullptr;
    std::int32_t* status = nullptr;
    std::int64_t* bounds = nullptr;
    bool integer = true;
    bool pinned = false;
    // the triangular wire form instead (pack_compact): node_off, adj_off,
    // u16 loads, adjacency bits; num / den / edge_off / edges unused
    bool tri = false;
    std::uint32_t *adj_off = nullptr, *adj = nullptr;
    std::uint16_t* ln16 = nullptr;
    struct Store;
    std::shared_ptr<Store> store;  // the arena lease or the heap block
    ds_dag_batch view() const {
        return ds_dag_batch{n_dags, node_off, edge_off, num, integer ? nullptr : den, edges};
    }
    ds_dag_batch_tri view_tri() const { return ds_dag_batch_tri{n_dags, node_off, adj_off, ln16, adj}; }
};

Packed pack(const std::vector<const DagTask*>& tasks, bool with_results = false);
// The triangular wire form when every task fits it (<= 64 nodes, integer
// loads < 2^16, local order topological: ~5x fewer bytes over PCIe, read by
// the device's fast path as is), else pack().
Packed pack_compact(const std::vector<const DagTask*>& tasks, bool with_results = false);
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

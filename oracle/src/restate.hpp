// TEST INFRASTRUCTURE — oracle restatement of the reference's hot path.
//
// An independent re-statement (flat arrays + word bitmasks instead of the
// reference's std::map/std::set/boost::dynamic_bitset) of:
//   exec_model.cpp:7-23            exec_time, max_parallelism
//   dag.cpp:22-138, 179-236        DagTask::make and its queries
//   division.cpp:10-126            build_blocks, local_paths, build_groups
//   scheduler.cpp:35-116, 175-427  apportion / scale_parallelism / schedule
//   analysis.cpp:11-99             the five bounds and analyze
//   generator.cpp:9-108            generate / generate_corpus (same RNG order)
//   experiment.cpp:27-79           method_bound / evaluate_corpus
// Every function cites the reference lines it follows. Exceptions mirror the
// reference's types so the C wrapper maps them to the same DS_* codes.
#pragma once

#include "q.hpp"

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
    int code;
    ValidationError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Platform {
    int M = 1;
    Q tmin = Q(1);
};

void check_platform(const Platform& p);
Q exec_time(const Q& load, long long m, const Platform& p);
int max_par(const Q& load, const Platform& p);

using Bits = std::vector<uint64_t>;

// Immutable DAG over local indices 0..n-1 (index order == id order).
struct Dag {
    int n = 0;
    std::vector<Q> load;
    std::vector<std::vector<int>> pred, succ;  // ascending indices
    std::vector<Bits> anc, desc;
    std::vector<Q> wanc;
    std::vector<int> topo;
    std::vector<std::pair<int, int>> edges;  // sorted, deduplicated
    int words() const { return (n + 63) / 64; }
};

// DagTask::make over local indices; throws ValidationError with the DS code.
Dag make_dag(std::vector<Q> loads, std::vector<std::pair<long long, long long>> edges,
             const Q& min_load);

std::vector<int> join_nodes(const Dag& g);
std::vector<std::vector<int>> build_blocks(const Dag& g, std::vector<int>* residual_flag = nullptr);
std::vector<std::vector<int>> local_paths(const Dag& g, const std::vector<int>& block);
std::vector<std::vector<int>> build_groups(const Dag& g, const Platform& p);

struct Ent {  // EntityId
    int origin = 0;
    int gen = 0;
    int part = 0;  // 0 whole, 1 parallel, 2 residual
};
bool operator<(const Ent& a, const Ent& b);
bool operator==(const Ent& a, const Ent& b);
std::string ent_str(const Ent& e);

struct Member {
    Ent e;
    Q load;
    int m;
    Q exec;
};
struct Launch {
    Ent e;
    int m;
    Q dur;
};
struct Group {
    int index;
    std::vector<Member> members;
    int spare;
    Q spare_cap;
    Q resp;
    Ent bottleneck;
    std::vector<Launch> launches;
};
struct Seg {
    Ent src, par, res;
    Q par_load, res_load;
    int group;
};
struct Record {
    Ent e;
    Q load;
    int m;
    Q exec;
    int group;
    bool launched;
    std::vector<Ent> preds;
};
struct Scheme {
    Platform plat;
    std::vector<Group> groups;
    std::vector<Seg> segs;
    std::vector<std::pair<Ent, Ent>> extra;
    std::vector<Record> ents;
};

std::vector<int> apportion(const std::vector<Q>& loads, const std::vector<int>& caps,
                           const Platform& p);
Scheme schedule(const Dag& g, const Platform& p);

Q proposed_bound(const Scheme& s);
Q greedy_bound(const Dag& g, const Platform& p);
Q greedy_unaware_bound(const Dag& g, const Platform& p);
Q graham_para_bound(const Dag& g, const Platform& p);
Q lower_bound(const Dag& g, const Platform& p);

struct GenCfg {
    int depth_min = 5, depth_max = 8, max_width = 8;
    Q avg_load = Q(20);
    double jitter = 0.5, density = 0.2;
    uint64_t seed = 1;
    bool integer_loads = true, exact_mean = false;
    Q tmin = Q(1);
};
Dag generate(const GenCfg& c);

std::string scheme_json(const Scheme& s);

}  // namespace orc

// Drives the kept C++ API (include/dagsched/*.hpp, libdagsched_cpp.so) the way
// a reference user would, and prints the results as JSON for
// tests/test_gpu_cpp_api.py to compare with the reference's golden outputs.
#include "dagsched/analysis.hpp"
#include "dagsched/division.hpp"
#include "dagsched/experiment.hpp"
#include "dagsched/generator.hpp"
#include "dagsched/scheduler.hpp"

#include <cstdio>
#include <iostream>
#include <sstream>

using namespace dagsched;

namespace {
std::string q(const Rational& r) { return "\"" + format_exact(r) + "\""; }
std::string e(const EntityId& id) { return "\"" + to_string(id) + "\""; }

std::string scheme_json(const ScheduleScheme& s) {
    std::ostringstream o;
    o << "{\"platform\": {\"sm_count\": " << s.platform.sm_count << ", \"t_min\": " << q(s.platform.t_min)
      << "}, \"groups\": [";
    for (std::size_t i = 0; i < s.groups.size(); ++i) {
        const GroupPlan& g = s.groups[i];
        o << (i ? ", " : "") << "{\"index\": " << g.index << ", \"members\": [";
        for (std::size_t k = 0; k < g.members.size(); ++k)
            o << (k ? ", " : "") << "{\"entity\": " << e(g.members[k].entity) << ", \"load\": " << q(g.members[k].load)
              << ", \"parallelism\": " << g.members[k].parallelism << ", \"exec_time\": " << q(g.members[k].exec) << "}";
        o << "], \"spare_sms\": " << g.spare_sms << ", \"spare_capacity\": " << q(g.spare_capacity)
          << ", \"response\": " << q(g.response) << ", \"bottleneck\": " << e(g.bottleneck) << ", \"launches\": [";
        for (std::size_t k = 0; k < g.launches.size(); ++k)
            o << (k ? ", " : "") << "{\"entity\": " << e(g.launches[k].entity) << ", \"parallelism\": "
              << g.launches[k].parallelism << ", \"duration\": " << q(g.launches[k].duration) << "}";
        o << "]}";
    }
    o << "], \"segmentations\": [";
    for (std::size_t i = 0; i < s.segmentations.size(); ++i) {
        const auto& x = s.segmentations[i];
        o << (i ? ", " : "") << "{\"source\": " << e(x.source) << ", \"parallel\": " << e(x.parallel)
          << ", \"residual\": " << e(x.residual) << ", \"parallel_load\": " << q(x.parallel_load)
          << ", \"residual_load\": " << q(x.residual_load) << ", \"group\": " << x.group << "}";
    }
    o << "], \"extra_deps\": [";
    for (std::size_t i = 0; i < s.extra_deps.size(); ++i)
        o << (i ? ", " : "") << "[" << e(s.extra_deps[i].first) << ", " << e(s.extra_deps[i].second) << "]";
    o << "], \"entities\": [";
    for (std::size_t i = 0; i < s.entities.size(); ++i) {
        const auto& r = s.entities[i];
        o << (i ? ", " : "") << "{\"id\": " << e(r.id) << ", \"load\": " << q(r.load) << ", \"parallelism\": "
          << r.parallelism << ", \"exec_time\": " << q(r.exec) << ", \"group\": " << r.group
          << ", \"launched\": " << (r.launched ? "true" : "false") << ", \"preds\": [";
        for (std::size_t k = 0; k < r.preds.size(); ++k) o << (k ? ", " : "") << e(r.preds[k]);
        o << "]}";
    }
    o << "]}";
    return o.str();
}

DagTask fig2() {  // paper Fig. 2, make_example_task (test_fixtures.hpp:12-21): ids 1..7
    return DagTask::make({{1, 1}, {2, 4}, {3, 3}, {4, 3}, {5, 2}, {6, 2}, {7, 1}},
                         {{1, 2}, {1, 3}, {1, 4}, {3, 5}, {4, 5}, {4, 6}, {2, 7}, {5, 7}, {6, 7}});
}
DagTask fan() {
    std::vector<DagNode> nodes{{0, 1}};
    std::vector<std::pair<NodeId, NodeId>> edges;
    for (NodeId i = 1; i <= 8; ++i) {
        nodes.push_back({i, 20});
        edges.push_back({0, i});
        edges.push_back({i, 9});
    }
    nodes.push_back({9, 1});
    return DagTask::make(nodes, edges);
}
}  // namespace

int main() {
    std::cout << "{\"fixtures\": [";
    struct Case {
        const char* name;
        DagTask t;
        int M;
    };
    std::vector<Case> cases{{"fig2", fig2(), 6}, {"fig2", fig2(), 8}, {"fig2", fig2(), 148},
                            {"c1_fan_8_20_1", fan(), 148}, {"c1_fan_8_20_1", fan(), 32}};
    for (std::size_t i = 0; i < cases.size(); ++i) {
        const Platform p{cases[i].M, Rational(1)};
        const MakespanReport r = analyze(cases[i].t, p);
        const BalancedGroupList g = build_groups(cases[i].t, p);
        std::cout << (i ? ", " : "") << "{\"name\": \"" << cases[i].name << "\", \"sm_count\": " << cases[i].M
                  << ", \"proposed\": " << q(r.proposed) << ", \"greedy\": " << q(r.greedy)
                  << ", \"greedy_unaware\": " << q(r.greedy_unaware) << ", \"graham_para\": " << q(r.graham_para)
                  << ", \"lower\": " << q(r.lower) << ", \"n_div_groups\": " << g.groups.size()
                  << ", \"bound_from_scheme\": " << q(dag_makespan_bound(schedule(cases[i].t, p)))
                  << ", \"scheme\": " << scheme_json(schedule(cases[i].t, p)) << "}";
    }
    GenConfig cfg;  // generate_corpus(GenConfig{}, seed 1, 1000) = tests/golden/corpus_default.npz
    const std::vector<DagTask> corpus = generate_corpus(cfg, 1000);
    const auto rows = evaluate_corpus(corpus, Platform{148, Rational(1)},
                                      {Method::proposed, Method::greedy, Method::greedy_unaware, Method::graham_para},
                                      true);
    std::cout << "], \"corpus_M148\": [";
    for (std::size_t i = 0; i < rows.size(); ++i) {
        std::cout << (i ? ", " : "") << "[";
        for (std::size_t k = 0; k < rows[i].size(); ++k) std::cout << (k ? ", " : "") << q(rows[i][k]);
        std::cout << "]";
    }
    std::cout << "]}\n";
    return 0;
}

// Division / scaling / candidate dump over the kept C++ API — the SAME source
// compiles against the reference's headers and library (oracle/_ref:
// ref_division_dump, which writes tests/golden/division.json) and against
// this repo's include/dagsched (libdagsched_cpp.so: api_division_dump), so the
// two outputs can be compared field by field. Covers build_blocks,
// local_paths, build_groups (division.cpp:10-126), scale_parallelism and
// parallel_candidates (scheduler.cpp:99-146) on hand-built tasks (the SPEC's
// known answers) and on generated corpora at
// several M. `--host-only` skips build_groups (the device call) and derives
// the groups that scale_parallelism / parallel_candidates take from a
// golden file instead: argv[2].
#include "dagsched/division.hpp"
#include "dagsched/generator.hpp"
#include "dagsched/scheduler.hpp"

#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <set>
#include <sstream>
#include <string>
#include <vector>

using namespace dagsched;

namespace {

std::string ids(const std::vector<NodeId>& v) {
    std::ostringstream o;
    o << "[";
    for (std::size_t i = 0; i < v.size(); ++i) o << (i ? ", " : "") << v[i];
    o << "]";
    return o.str();
}

DagTask fig2() {  // make_example_task (test_fixtures.hpp:12-21)
    return DagTask::make({{1, 1}, {2, 4}, {3, 3}, {4, 3}, {5, 2}, {6, 2}, {7, 1}},
                         {{1, 2}, {1, 3}, {1, 4}, {3, 5}, {4, 5}, {4, 6}, {2, 7}, {5, 7}, {6, 7}});
}
DagTask chain3() { return DagTask::make({{10, 2}, {11, 3}, {12, 1}}, {{10, 11}, {11, 12}}); }
DagTask diamond(int s, int a, int b, int t) {
    return DagTask::make({{0, s}, {1, a}, {2, b}, {3, t}}, {{0, 1}, {0, 2}, {1, 3}, {2, 3}});
}
DagTask fan(int k, int mid, int end) {
    std::vector<DagNode> nodes{{0, end}};
    std::vector<std::pair<NodeId, NodeId>> edges;
    for (NodeId i = 1; i <= NodeId(k); ++i) {
        nodes.push_back({i, mid});
        edges.push_back({0, i});
        edges.push_back({i, NodeId(k + 1)});
    }
    nodes.push_back({NodeId(k + 1), end});
    return DagTask::make(nodes, edges);
}
// groups {a,b}, loads 4,2,2 inside one fork
DagTask fork3() {
    return DagTask::make({{0, 1}, {1, 4}, {2, 2}, {3, 2}, {4, 1}}, {{0, 1}, {0, 2}, {0, 3}, {1, 4}, {2, 4}, {3, 4}});
}

struct Case {
    std::string name;
    DagTask task;
    int M;
};

// groups from a golden line "G <case index> <g> <id> <id> ...", for --host-only
std::vector<std::vector<std::vector<NodeId>>> read_groups(const char* path, std::size_t n_cases) {
    std::vector<std::vector<std::vector<NodeId>>> out(n_cases);
    std::ifstream f(path);
    std::string line;
    while (std::getline(f, line)) {
        std::istringstream in(line);
        std::string tag;
        std::size_t c, g;
        if (!(in >> tag >> c >> g) || tag != "G" || c >= n_cases) continue;
        if (out[c].size() <= g) out[c].resize(g + 1);
        NodeId v;
        while (in >> v) out[c][g].push_back(v);
    }
    return out;
}

}  // namespace

int main(int argc, char** argv) {
    const bool host_only = argc > 2 && std::strcmp(argv[1], "--host-only") == 0;
    // --big: only generated DAGs of ~190-940 nodes (the paper's P = 32 sweep
    // and deeper), compared live against the reference's build of this file
    const bool big = argc > 1 && std::strcmp(argv[1], "--big") == 0;
    std::vector<Case> cases;
    if (big) {
        GenConfig mid;
        mid.seed = 700;
        mid.max_width = 32;
        mid.depth_min = 16;
        mid.depth_max = 26;
        const auto a = generate_corpus(mid, 6);
        for (int M : {8, 32, 148})
            for (std::size_t i = 0; i < a.size(); ++i) cases.push_back({"p32_seed" + std::to_string(700 + i), a[i], M});
        GenConfig huge = mid;
        huge.seed = 800;
        huge.max_width = 48;
        huge.depth_min = 26;
        huge.depth_max = 34;
        const auto h = generate_corpus(huge, 3);
        for (int M : {8, 148})
            for (std::size_t i = 0; i < h.size(); ++i) cases.push_back({"p48_seed" + std::to_string(800 + i), h[i], M});
    }
    if (!big)
        for (int M : {3, 4, 5, 6, 8, 148}) cases.push_back({"fig2", fig2(), M});
    if (!big) {
    cases.push_back({"chain3", chain3(), 4});
    cases.push_back({"diamond_1_5_2_1", diamond(1, 5, 2, 1), 4});
    cases.push_back({"diamond_1_5_2_1", diamond(1, 5, 2, 1), 148});
    cases.push_back({"fan_8_20_1", fan(8, 20, 1), 148});
    cases.push_back({"fan_8_20_1", fan(8, 20, 1), 32});
    cases.push_back({"fan_12_7_3", fan(12, 7, 3), 5});
    cases.push_back({"fork3", fork3(), 6});
    {
        GenConfig cfg;  // GenConfig{} defaults (generator.hpp:16-25)
        cfg.seed = 1;
        const auto corpus = generate_corpus(cfg, 60);
        for (int M : {4, 8, 32, 148})
            for (std::size_t i = 0; i < corpus.size(); ++i)
                cases.push_back({"default_seed" + std::to_string(1 + i), corpus[i], M});
        GenConfig wide;  // many heads per block: Rule 1's top-M cut at small M
        wide.seed = 300;
        wide.max_width = 24;
        wide.depth_min = 6;
        wide.depth_max = 10;
        wide.avg_load = Rational(40);
        const auto w = generate_corpus(wide, 20);
        for (int M : {3, 8, 148})
            for (std::size_t i = 0; i < w.size(); ++i) cases.push_back({"wide_seed" + std::to_string(300 + i), w[i], M});
        GenConfig heavy;  // oversized heads: Rule 2
        heavy.seed = 100;
        heavy.avg_load = Rational(200);
        const auto h = generate_corpus(heavy, 20);
        for (int M : {8, 148})
            for (std::size_t i = 0; i < h.size(); ++i) cases.push_back({"heavy_seed" + std::to_string(100 + i), h[i], M});
    }
    }
    std::vector<std::vector<std::vector<NodeId>>> given;
    if (host_only) given = read_groups(argv[2], cases.size());

    std::cout << "{\"cases\": [\n";
    for (std::size_t c = 0; c < cases.size(); ++c) {
        const DagTask& t = cases[c].task;
        const Platform p{cases[c].M, Rational(1)};
        std::cout << (c ? ",\n" : "") << "{\"name\": \"" << cases[c].name << "\", \"sm_count\": " << cases[c].M;
        const auto blocks = build_blocks(t);
        std::cout << ", \"blocks\": [";
        for (std::size_t b = 0; b < blocks.size(); ++b) {
            std::cout << (b ? ", " : "") << "{\"join\": ";
            if (blocks[b].join) std::cout << *blocks[b].join;
            else std::cout << "null";
            std::cout << ", \"members\": " << ids(blocks[b].members) << ", \"paths\": [";
            const auto lp = local_paths(t, blocks[b]);
            for (std::size_t k = 0; k < lp.paths.size(); ++k) std::cout << (k ? ", " : "") << ids(lp.paths[k]);
            std::cout << "]}";
        }
        std::cout << "]";
        std::vector<std::vector<NodeId>> groups;
        if (host_only) {
            groups = given[c];
        } else {
            groups = build_groups(t, p).groups;
            std::cout << ", \"groups\": [";
            for (std::size_t g = 0; g < groups.size(); ++g) std::cout << (g ? ", " : "") << ids(groups[g]);
            std::cout << "]";
        }
        // per division group: scale_parallelism, and parallel_candidates with
        // released = every node whose predecessors all lie in earlier groups
        // (SPEC.md:274), and with released = V
        std::set<NodeId> earlier, all;
        for (const DagNode& v : t.nodes()) all.insert(v.id);
        std::cout << ", \"scale\": [";
        for (std::size_t g = 0; g < groups.size(); ++g) {
            const auto m = scale_parallelism(groups[g], t, p);
            std::cout << (g ? ", " : "") << "[";
            bool first = true;
            for (const auto& [v, q] : m) {
                std::cout << (first ? "" : ", ") << "[" << v << ", " << q << "]";
                first = false;
            }
            std::cout << "]";
        }
        std::cout << "], \"cands\": [";
        for (std::size_t g = 0; g < groups.size(); ++g) {
            std::set<NodeId> released;
            for (const DagNode& v : t.nodes()) {
                bool ok = !earlier.count(v.id);
                for (NodeId u : t.predecessors(v.id)) ok &= earlier.count(u) > 0;
                if (ok) released.insert(v.id);
            }
            std::cout << (g ? ", " : "") << "[" << ids(parallel_candidates(groups[g], t, released)) << ", "
                      << ids(parallel_candidates(groups[g], t, all)) << "]";
            earlier.insert(groups[g].begin(), groups[g].end());
        }
        std::cout << "]}";
        if (!host_only) {
            for (std::size_t g = 0; g < groups.size(); ++g) {
                std::cerr << "G " << c << " " << g;
                for (NodeId v : groups[g]) std::cerr << " " << v;
                std::cerr << "\n";
            }
        }
    }
    std::cout << "\n]}\n";
    return 0;
}

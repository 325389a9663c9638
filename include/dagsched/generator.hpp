// dagsched_b200 — kept C++ API: the layered random DAG generator (§5.1).
// GenConfig fields and generate/generate_corpus of the reference's
// generator.hpp:15-33, bit-identical output (host, ds_corpus_generate).
#pragma once

#include "dagsched/dag.hpp"

#include <cstdint>
#include <vector>

namespace dagsched {

struct GenConfig {
    int depth_min = 5;
    int depth_max = 8;
    int max_width = 8;  // P
    Rational avg_load = Rational(20);
    double load_jitter = 0.5;
    double edge_density = 0.2;
    std::uint64_t seed = 1;
    bool integer_loads = true;
    bool exact_mean = false;
    Rational t_min = Rational(1);

    void check() const;  // std::invalid_argument on a bad configuration
};

DagTask generate(const GenConfig& config);
std::vector<DagTask> generate_corpus(const GenConfig& config, int count);  // seeds seed, seed+1, ...

}  // namespace dagsched

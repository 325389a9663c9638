// C++ API latency / throughput — the SAME source compiles against the
// reference's headers and library (oracle/_ref/ref_api_bench: the reference's
// own CPU code) and against this repo's kept API (api_bench: the GPU path
// behind include/dagsched), so the two JSON lines measure the same calls:
//
//   c1_*        analyze() / schedule() of the C1 fork-join task (make_fan(8,
//               20, 1), tests/test_fixtures.hpp:43-53) at M = 148: one call's
//               latency, median and p99 over `reps` calls after warm-up.
//   corpus_*    evaluate_corpus(corpus, M = 148, all four methods, parallel)
//               + building the Rational results (experiment.hpp:51): the
//               reference's batch boundary end to end, on generate_corpus(
//               GenConfig{}, n) (generation timed separately, excluded).
//
// usage: api_bench [n_corpus=100000] [reps=200]
#include "dagsched/analysis.hpp"
#include "dagsched/experiment.hpp"
#include "dagsched/generator.hpp"
#include "dagsched/scheduler.hpp"

#ifdef DS_API_BENCH_RAW  // this repo's build: also time the bare C-ABI calls
#include "dagsched_b200.h"
#endif

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

using namespace dagsched;
using Clock = std::chrono::steady_clock;

namespace {

DagTask make_fan(int n, Rational mid, Rational end) {
    std::vector<DagNode> nodes{{0, end}};
    std::vector<std::pair<NodeId, NodeId>> edges;
    for (int i = 1; i <= n; ++i) {
        nodes.push_back({static_cast<NodeId>(i), mid});
        edges.push_back({0, static_cast<NodeId>(i)});
        edges.push_back({static_cast<NodeId>(i), static_cast<NodeId>(n + 1)});
    }
    nodes.push_back({static_cast<NodeId>(n + 1), end});
    return DagTask::make(std::move(nodes), std::move(edges));
}

double us_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::micro>(Clock::now() - t0).count();
}

struct Lat {
    double p50, p99, mean;
};

template <class F>
Lat latency(int reps, F&& f) {
    for (int i = 0; i < 10; ++i) f();  // warm-up (device init, first allocations)
    std::vector<double> us;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = Clock::now();
        f();
        us.push_back(us_since(t0));
    }
    double sum = 0;
    for (double x : us) sum += x;
    std::sort(us.begin(), us.end());
    return Lat{us[us.size() / 2], us[std::min(us.size() - 1, us.size() * 99 / 100)], sum / us.size()};
}

}  // namespace

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 100000;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 200;
    const Platform p148{148, Rational(1)};
    const DagTask c1 = make_fan(8, Rational(20), Rational(1));
    Rational sink;
    const Lat la = latency(reps, [&] { sink = analyze(c1, p148).proposed; });
    const std::string proposed = format_exact(sink);
    std::size_t groups = 0;
    const Lat ls = latency(reps, [&] { groups = schedule(c1, p148).groups.size(); });

    std::string raw = "";
#ifdef DS_API_BENCH_RAW
    {  // the C-ABI calls alone on the packed C1 task (no DagTask packing / materialisation)
        const uint32_t no[2] = {0, 10}, eo[2] = {0, 16};
        int64_t ln[10] = {1, 20, 20, 20, 20, 20, 20, 20, 20, 1};
        uint32_t ed[16];
        for (int i = 1; i <= 8; ++i) ed[i - 1] = (0u << 16) | uint32_t(i), ed[7 + i] = (uint32_t(i) << 16) | 9u;
        std::sort(ed, ed + 16);
        const ds_dag_batch b{1, no, eo, ln, nullptr, ed};
        const ds_platform pl{148, 0, 1, 1};
        int32_t st = 0;
        int64_t bounds[10];
        uint16_t ne = 0, ng = 0, nd = 0;
        int16_t nb[10], ndg[10];
        ds_entity_rec ents[20];
        ds_group_rec grps[10];
        ds_results r{&st, bounds, nullptr};
        ds_scheme_out so{&st, &ne, &ng, &nd, nb, ndg, ents, grps, bounds};
        const Lat ra = latency(reps, [&] { ds_analyze_batch(&b, &pl, DS_M_ALL, &r, 0, nullptr, 0); });
        const Lat rs = latency(reps, [&] { ds_schedule_batch(&b, &pl, &so, 0); });
        char buf[256];
        std::snprintf(buf, sizeof buf, "\"c1_raw_ds_analyze_batch_us\": {\"p50\": %.2f, \"p99\": %.2f}, "
                      "\"c1_raw_ds_schedule_batch_us\": {\"p50\": %.2f, \"p99\": %.2f}, ", ra.p50, ra.p99, rs.p50, rs.p99);
        raw = buf;
    }
#endif
    GenConfig cfg;
    auto t0 = Clock::now();
    const std::vector<DagTask> corpus = generate_corpus(cfg, n);
    const double gen_s = us_since(t0) / 1e6;
    const std::vector<Method> methods{Method::proposed, Method::greedy, Method::greedy_unaware, Method::graham_para};
    evaluate_corpus(std::vector<DagTask>(corpus.begin(), corpus.begin() + std::min<std::size_t>(corpus.size(), 1000)),
                    p148, methods, true);  // warm-up
    double best = 1e30;
    std::string check;
    for (int r = 0; r < 3; ++r) {
        t0 = Clock::now();
        const auto rows = evaluate_corpus(corpus, p148, methods, true);
        best = std::min(best, us_since(t0) / 1e6);
        unsigned long long h = 1469598103934665603ull;  // FNV-1a over every bound's exact text
        for (const auto& row : rows)
            for (const Rational& q : row)
                for (char c : format_exact(q) + ";") h = (h ^ (unsigned char)c) * 1099511628211ull;
        check = std::to_string(h);
    }
    std::printf("{%s\"c1_analyze_us\": {\"p50\": %.2f, \"p99\": %.2f, \"mean\": %.2f}, "
                "\"c1_schedule_us\": {\"p50\": %.2f, \"p99\": %.2f, \"mean\": %.2f}, \"c1_proposed\": \"%s\", "
                "\"c1_groups\": %zu, \"corpus_dags\": %d, \"corpus_generate_s\": %.3f, "
                "\"corpus_evaluate_s\": %.4f, \"corpus_dags_per_s\": %.1f, \"corpus_checksum\": \"%s\", "
                "\"reps\": %d}\n",
                raw.c_str(), la.p50, la.p99, la.mean, ls.p50, ls.p99, ls.mean, proposed.c_str(), groups, n, gen_s, best,
                n / best, check.c_str(), reps);
    return 0;
}

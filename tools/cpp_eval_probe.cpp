// Phase timing of the kept C++ evaluate_corpus on 1M generated DAGs:
// DagTask packing, the C-ABI call (pageable vs pinned), Rational results.
//   make -C . tools/cpp_eval_probe (see tools/gpu_cpp_eval.sh)
#include "dagsched/experiment.hpp"
#include "dagsched/generator.hpp"
#include "dagsched_b200.h"
#include "device.hpp"

#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

using namespace dagsched;
using Clock = std::chrono::steady_clock;
static double ms(Clock::time_point a) { return std::chrono::duration<double, std::milli>(Clock::now() - a).count(); }

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 1000000;
    GenConfig cfg;
    auto t = Clock::now();
    const auto corpus = generate_corpus(cfg, n);
    std::printf("generate_corpus %.1f ms\n", ms(t));
    const Platform p{148, Rational(1)};
    const std::vector<Method> methods{Method::proposed, Method::greedy, Method::greedy_unaware, Method::graham_para};
    evaluate_corpus(std::vector<DagTask>(corpus.begin(), corpus.begin() + 1000), p, methods, true);
    for (int r = 0; r < 3; ++r) {
        t = Clock::now();
        const auto rows = evaluate_corpus(corpus, p, methods, true);
        std::printf("evaluate_corpus total %.1f ms\n", ms(t));
    }
    std::vector<const DagTask*> ptrs;
    for (const auto& c : corpus) ptrs.push_back(&c);
    t = Clock::now();
    {
        const detail::Packed pk = detail::pack(ptrs, true);
        std::printf("pack %.1f ms (integer %d, pinned %d)\n", ms(t), int(pk.integer), int(pk.pinned));
        const ds_dag_batch b = pk.view();
        const ds_platform pl = detail::platform_of(p);
        ds_results r{pk.status, pk.bounds, nullptr};
        int dev = 0;
        for (int k = 0; k < 3; ++k) {
            t = Clock::now();
            ds_analyze_batch_multi(&b, &pl, 0xF, &r, &dev, 1);
            std::printf("ds_analyze_batch_multi (packed block) %.1f ms\n", ms(t));
        }
    }
    std::vector<int64_t> bounds(size_t(n) * 10, 1);
    t = Clock::now();
    std::vector<std::vector<Rational>> out(n);
    detail::parallel_for(n, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            out[i].reserve(4);
            for (int m = 0; m < 4; ++m)
                out[i].push_back(Rational::reduced(BigInt(bounds[10 * i + 2 * m]), BigInt(bounds[10 * i + 2 * m + 1])));
        }
    });
    std::printf("results %.1f ms\n", ms(t));
    t = Clock::now();
    { auto tmp = std::move(out); }
    std::printf("free results %.1f ms\n", ms(t));
    return 0;
}

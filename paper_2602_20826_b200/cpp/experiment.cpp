// Kept C++ API — the batch boundary: evaluate_corpus on the GPU(s).
#include "dagsched/experiment.hpp"

#include "device.hpp"

namespace dagsched {

std::string method_name(Method m) {
    switch (m) {
        case Method::proposed: return "proposed";
        case Method::greedy: return "greedy";
        case Method::greedy_unaware: return "greedy_unaware";
        case Method::graham_para: return "graham_para";
    }
    throw std::logic_error("unknown method");
}

std::vector<std::vector<Rational>> evaluate_corpus(const std::vector<DagTask>& corpus, const Platform& platform,
                                                   const std::vector<Method>& methods, bool /*parallel*/) {
    std::vector<const DagTask*> ptrs;
    for (const DagTask& t : corpus) ptrs.push_back(&t);
    const detail::Packed p = detail::pack(ptrs);
    const ds_dag_batch b = p.view();
    const ds_platform pl = detail::platform_of(platform);
    uint32_t mask = 0;
    for (Method m : methods) mask |= 1u << int(m);  // Method order == DS_BOUND_* slots
    std::vector<int32_t> st(corpus.size());
    std::vector<int64_t> bounds(corpus.size() * 10);
    ds_results r{st.data(), bounds.data(), nullptr};
    const std::vector<int> devs = detail::devices();
    detail::check(ds_analyze_batch_multi(&b, &pl, mask, &r, devs.data(), int(devs.size())));
    for (std::size_t i = 0; i < corpus.size(); ++i)  // the first failing task, in order
        if (st[i] != DS_OK) detail::raise(st[i], "evaluate_corpus: task " + std::to_string(i));
    std::vector<std::vector<Rational>> out(corpus.size());
    detail::parallel_for(corpus.size(), [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            out[i].reserve(methods.size());
            for (Method m : methods) {
                const int k = int(m);
                out[i].push_back(
                    Rational::reduced(BigInt(bounds[10 * i + 2 * k]), BigInt(bounds[10 * i + 2 * k + 1])));
            }
        }
    });
    return out;
}

}  // namespace dagsched

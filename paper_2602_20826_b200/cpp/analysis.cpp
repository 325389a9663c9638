// Kept C++ API — bounds. The per-task bounds are one device launch of K1
// (ds_analyze_batch); group sums are host arithmetic over a ScheduleScheme.
#include "dagsched/analysis.hpp"

#include "device.hpp"

namespace dagsched {

namespace {
Rational bound_of(const DagTask& task, const Platform& platform, int slot) {
    const detail::Packed p = detail::pack({&task});
    const ds_dag_batch b = p.view();
    const ds_platform pl = detail::platform_of(platform);
    int32_t st = 0;
    int64_t bounds[10] = {};
    ds_results r{&st, bounds, nullptr};
    detail::check(ds_analyze_batch(&b, &pl, 1u << slot, &r, detail::devices().front(), nullptr, 0));
    detail::raise(st, "bound");
    return Rational::reduced(BigInt(bounds[2 * slot]), BigInt(bounds[2 * slot + 1]));
}
}  // namespace

Rational group_response_time(const GroupPlan& plan) {
    Rational r;
    for (const MemberPlan& m : plan.members)
        if (m.exec > r) r = m.exec;
    return r;
}

Rational dag_makespan_bound(const ScheduleScheme& scheme) {
    Rational t;
    for (const GroupPlan& g : scheme.groups) t += g.response;
    return t;
}

Rational greedy_bound(const DagTask& t, const Platform& p) { return bound_of(t, p, DS_BOUND_GREEDY); }
Rational greedy_unaware_bound(const DagTask& t, const Platform& p) { return bound_of(t, p, DS_BOUND_GREEDY_UNAWARE); }
Rational graham_para_bound(const DagTask& t, const Platform& p) { return bound_of(t, p, DS_BOUND_GRAHAM_PARA); }
Rational lower_bound(const DagTask& t, const Platform& p) { return bound_of(t, p, DS_BOUND_LOWER); }

// One device pass (ds_schedule_batch: K1 in detail mode) yields the schedule
// and all five bounds; the reference's analyze() runs schedule() and then the
// four baseline bounds (analysis.cpp:83-99).
MakespanReport analyze(const DagTask& task, const Platform& platform) {
    std::vector<int64_t> bounds;
    const ScheduleScheme s =
        std::move(detail::schedule_ptrs({&task}, platform, detail::devices().front(), &bounds).front());
    auto q = [&](int k) { return Rational::reduced(BigInt(bounds[2 * k]), BigInt(bounds[2 * k + 1])); };
    MakespanReport rep;
    for (const GroupPlan& g : s.groups) rep.per_group_response.push_back(g.response);
    rep.proposed = dag_makespan_bound(s);
    rep.greedy = q(DS_BOUND_GREEDY);
    rep.greedy_unaware = q(DS_BOUND_GREEDY_UNAWARE);
    rep.graham_para = q(DS_BOUND_GRAHAM_PARA);
    rep.lower = q(DS_BOUND_LOWER);
    rep.normalized["proposed"] = rep.proposed / rep.greedy_unaware;
    rep.normalized["greedy"] = rep.greedy / rep.greedy_unaware;
    rep.normalized["greedy_unaware"] = Rational(1);
    rep.normalized["graham_para"] = rep.graham_para / rep.greedy_unaware;
    return rep;
}

}  // namespace dagsched

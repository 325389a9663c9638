// Kept C++ API — the batch boundary (evaluate_corpus on the GPU(s)) and the
// sweep drivers over it (include/dagsched/experiment.hpp; the reference's
// experiment.cpp:52-307 semantics: same sweeps, seeds, reductions, CSVs).
#include "dagsched/experiment.hpp"

#include "bigfrac.hpp"
#include "dagsched/scheduler.hpp"
#include "dagsched/simulator.hpp"
#include "dagsched/task_io.hpp"
#include "device.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <ostream>
#include <stdexcept>

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

namespace {

std::string sweep_var_name(ExperimentSpec::SweepVar v) {
    switch (v) {
        case ExperimentSpec::SweepVar::sm_count: return "M";
        case ExperimentSpec::SweepVar::max_width: return "P";
        case ExperimentSpec::SweepVar::depth: return "V";
    }
    throw std::logic_error("unknown sweep variable");
}

uint32_t method_mask(const std::vector<Method>& methods) {
    uint32_t mask = 0;
    for (Method m : methods) mask |= 1u << int(m);  // Method order == DS_BOUND_* slots
    return mask;
}

// generate_corpus(cfg, n) straight into the packed batch form (the same
// bit-identical generator as generate_corpus, without building DagTasks)
struct GenBatch {
    void* h = nullptr;
    ds_dag_batch view{};
    GenBatch(const GenConfig& c, int count) {
        c.check();
        if (count < 1) throw std::invalid_argument("count must be >= 1");
        ds_gen_config g{c.depth_min, c.depth_max, c.max_width, c.integer_loads ? 1 : 0,
                        to_int64(numerator(c.avg_load)), to_int64(denominator(c.avg_load)), c.load_jitter,
                        c.edge_density, c.seed, to_int64(numerator(c.t_min)), to_int64(denominator(c.t_min)),
                        c.exact_mean ? 1 : 0, 0};
        detail::check(ds_corpus_generate(&g, count, DS_F_PINNED, &h));
        detail::check(ds_corpus_view(h, &view));
    }
    ~GenBatch() {
        if (h) ds_corpus_free(h);
    }
    GenBatch(const GenBatch&) = delete;
    GenBatch& operator=(const GenBatch&) = delete;
};

// generate()'s tasks are made with min_load = t_min (platform flag 0)
ds_platform generated_platform(const Platform& p) {
    p.check();
    return ds_platform{p.sm_count, 0, to_int64(numerator(p.t_min)), to_int64(denominator(p.t_min))};
}

Rational bound_at(const std::vector<int64_t>& b, std::size_t i, int slot) {
    return Rational::reduced(BigInt(b[10 * i + 2 * slot]), BigInt(b[10 * i + 2 * slot + 1]));
}

}  // namespace

std::vector<std::vector<Rational>> evaluate_corpus(const std::vector<DagTask>& corpus, const Platform& platform,
                                                   const std::vector<Method>& methods, bool /*parallel*/) {
    std::vector<const DagTask*> ptrs;
    ptrs.reserve(corpus.size());
    for (const DagTask& t : corpus) ptrs.push_back(&t);
    // inputs and result staging in one packed block (the pinned arena for a
    // large corpus), so both copy directions run at full PCIe rate
    const detail::Packed p = detail::pack_compact(ptrs, true);
    const ds_platform pl = detail::platform_of(platform);
    ds_results r{p.status, p.bounds, nullptr};
    const std::vector<int> devs = detail::devices();
    if (p.tri) {
        const ds_dag_batch_tri b = p.view_tri();
        detail::check(ds_analyze_batch_tri_multi(&b, &pl, method_mask(methods), &r, devs.data(), int(devs.size())));
    } else {
        const ds_dag_batch b = p.view();
        detail::check(ds_analyze_batch_multi(&b, &pl, method_mask(methods), &r, devs.data(), int(devs.size())));
    }
    for (std::size_t i = 0; i < corpus.size(); ++i)  // the first failing task, in order
        if (p.status[i] != DS_OK) detail::raise(p.status[i], "evaluate_corpus: task " + std::to_string(i));
    std::vector<std::vector<Rational>> out(corpus.size());
    const int64_t* bounds = p.bounds;
    detail::parallel_for(corpus.size(), [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            out[i].reserve(methods.size());
            for (Method m : methods) {
                const int k = int(m);
                out[i].push_back(Rational::reduced(BigInt(bounds[10 * i + 2 * k]), BigInt(bounds[10 * i + 2 * k + 1])));
            }
        }
    });
    return out;
}

// experiment.cpp:81-150: per sweep value a fresh corpus and one device pass
std::vector<ResultRow> run_experiment(const ExperimentSpec& spec) {
    if (spec.values.empty()) throw std::invalid_argument("no sweep values");
    if (spec.corpus_size < 1) throw std::invalid_argument("corpus_size must be >= 1");
    spec.base.check();
    spec.platform.check();
    std::vector<Method> methods = spec.methods;
    if (std::find(methods.begin(), methods.end(), spec.normalize_to) == methods.end())
        methods.push_back(spec.normalize_to);
    const int ref = int(spec.normalize_to);
    const std::vector<int> devs = detail::devices();
    std::vector<ResultRow> rows;
    for (long long value : spec.values) {
        GenConfig cfg = spec.base;
        Platform platform = spec.platform;
        switch (spec.sweep) {
            case ExperimentSpec::SweepVar::sm_count: platform.sm_count = int(value); break;
            case ExperimentSpec::SweepVar::max_width: cfg.max_width = int(value); break;
            case ExperimentSpec::SweepVar::depth: cfg.depth_min = cfg.depth_max = int(value); break;
        }
        const GenBatch gb(cfg, spec.corpus_size);
        const std::size_t n = std::size_t(spec.corpus_size);
        const ds_platform pl = generated_platform(platform);
        std::vector<int32_t> st(n);
        std::vector<int64_t> b(n * 10);
        ds_results r{st.data(), b.data(), nullptr};
        detail::check(ds_analyze_batch_multi(&gb.view, &pl, method_mask(methods), &r, devs.data(), int(devs.size())));
        for (std::size_t i = 0; i < n; ++i)
            if (st[i] != DS_OK) detail::raise(st[i], "run_experiment: task " + std::to_string(i));
        for (Method m : spec.methods) {
            detail::BigFrac norm_sum, abs_sum;
            std::vector<Rational> norms;
            norms.reserve(n);
            for (std::size_t i = 0; i < n; ++i) {
                const Rational x = bound_at(b, i, int(m));
                norms.push_back(x / bound_at(b, i, ref));
                norm_sum.add(norms.back());
                abs_sum.add(x);
            }
            norm_sum.div_int(n);
            abs_sum.div_int(n);
            ResultRow row;
            row.sweep_var = sweep_var_name(spec.sweep);
            row.sweep_value = value;
            row.method = m;
            bool exact = true;
            row.mean_norm = norm_sum.to_rational_or_truncated(exact);
            const double mean_d = to_double(row.mean_norm);
            double var = 0.0;
            for (const Rational& q : norms) {  // the reference's order of double accumulation
                const double d = to_double(q) - mean_d;
                var += d * d;
            }
            var /= double(n);
            row.std_norm = std::sqrt(var);
            row.mean_abs = abs_sum.to_rational_or_truncated(exact);
            row.n = spec.corpus_size;
            row.seed = cfg.seed;
            rows.push_back(std::move(row));
        }
    }
    return rows;
}

void write_csv(const std::vector<ResultRow>& rows, std::ostream& out) {
    out << "sweep_var,sweep_value,method,mean_norm,std_norm,mean_abs,n,seed\n";
    char buf[64];
    for (const ResultRow& r : rows) {
        std::snprintf(buf, sizeof(buf), "%.6f", r.std_norm);
        out << r.sweep_var << "," << r.sweep_value << "," << method_name(r.method) << ","
            << format_fixed(r.mean_norm, 6) << "," << buf << "," << format_fixed(r.mean_abs, 6) << "," << r.n << ","
            << r.seed << "\n";
    }
}

// experiment.cpp:163-240 on the device: K1 schedules + K4 simulations of
// every task at worst case and `samples` scaled runs (seeds config.seed +
// 7919 i + s), summary doubles reduced in the reference's order.
ValidationSummary run_validation(const GenConfig& config, int corpus_size, const Platform& platform, int samples,
                                 const Rational& scale_min, const Rational& scale_max, bool /*parallel*/) {
    config.check();
    platform.check();
    const GenBatch gb(config, corpus_size);
    const std::size_t n = std::size_t(corpus_size);
    const ds_platform pl = generated_platform(platform);
    std::vector<int32_t> st(n), viol(n);
    ds_validation sum{};
    detail::check(ds_validate_batch(&gb.view, &pl, samples, to_int64(numerator(scale_min)),
                                    to_int64(denominator(scale_min)), to_int64(numerator(scale_max)),
                                    to_int64(denominator(scale_max)), config.seed, st.data(), viol.data(), nullptr,
                                    nullptr, &sum, detail::devices().front()));
    for (std::size_t i = 0; i < n; ++i)
        if (st[i] != DS_OK) detail::raise(st[i], "run_validation: task " + std::to_string(i));
    ValidationSummary s;
    s.tasks = corpus_size;
    s.runs = corpus_size * (samples + 1);
    s.violations = int(sum.violations);
    s.mean_tightness_worst = sum.mean_tightness_worst;
    s.mean_tightness_scaled = sum.mean_tightness_scaled;
    // details for any violating task (never expected: Theorem 1), rebuilt
    // with the reference's wording from the same schedule and draws
    for (std::size_t i = 0; i < n; ++i) {
        if (viol[i] == 0) continue;
        const ds_dag_batch& v = gb.view;
        std::vector<DagNode> nodes;
        std::vector<std::pair<NodeId, NodeId>> edges;
        for (uint32_t k = v.node_off[i]; k < v.node_off[i + 1]; ++k)
            nodes.push_back(DagNode{k - v.node_off[i], Rational(BigInt(v.load_num[k]),
                                                                BigInt(v.load_den ? v.load_den[k] : 1))});
        for (uint32_t e = v.edge_off[i]; e < v.edge_off[i + 1]; ++e)
            edges.emplace_back(v.edges[e] >> 16, v.edges[e] & 0xffffu);
        const DagTask task = DagTask::make(std::move(nodes), std::move(edges), std::nullopt, config.t_min);
        const ScheduleScheme scheme = schedule(task, platform);
        const Rational bound = dag_makespan_bound(scheme);
        SimConfig sim;
        sim.platform = platform;
        std::string details;
        const SimTrace worst = simulate_scheme(task, scheme, sim);
        if (worst.makespan > bound)
            details += "task " + std::to_string(i) + ": worst-case makespan " + format_exact(worst.makespan) +
                       " > bound " + format_exact(bound) + "\n";
        for (int k = 0; k < samples; ++k) {
            sim.time_model.kind = TimeModel::Kind::scaled;
            sim.time_model.seed = config.seed + 7919 * i + std::uint64_t(k);
            sim.time_model.scale_min = scale_min;
            sim.time_model.scale_max = scale_max;
            const SimTrace t = simulate_scheme(task, scheme, sim);
            if (t.makespan > bound)
                details += "task " + std::to_string(i) + " sample " + std::to_string(k) + ": makespan " +
                           format_exact(t.makespan) + " > bound " + format_exact(bound) + "\n";
        }
        if (!details.empty()) s.violation_details.push_back(details);
    }
    return s;
}

// experiment.cpp:242-291: every (fixture, average load) variant at every M
// through one K1 schedule pass, one K1 bounds pass and one K6 pass (all runs)
std::vector<BenchCell> run_benchmarks(const std::vector<std::string>& fixture_paths, const std::vector<int>& sm_counts,
                                      const std::vector<long long>& avg_loads, int greedy_runs, std::uint64_t seed) {
    struct Variant {
        std::string name;
        long long avg;
        DagTask task;
    };
    std::vector<Variant> vars;
    for (const std::string& path : fixture_paths) {
        const DagTask base = read_task_file(path);
        const std::string name = std::filesystem::path(path).stem().string();
        for (long long avg : avg_loads) {
            std::vector<DagNode> nodes = base.nodes();  // fixtures carry unit loads
            for (DagNode& v : nodes) v.load *= Rational(avg, 1);
            vars.push_back(Variant{name, avg, DagTask::make(nodes, base.edges())});
        }
    }
    std::vector<const DagTask*> ptrs;
    for (const Variant& v : vars) ptrs.push_back(&v.task);
    const int dev = detail::devices().front();
    const detail::Packed p = detail::pack(ptrs);
    const ds_dag_batch b = p.view();
    const std::size_t nv = vars.size(), runs = std::size_t(std::max(0, greedy_runs));
    struct PerM {
        std::vector<ScheduleScheme> schemes;
        std::vector<int32_t> st, gst;
        std::vector<int64_t> bounds, gmk;
        std::string err;
    };
    std::vector<PerM> per(sm_counts.size());
    for (std::size_t k = 0; k < sm_counts.size(); ++k) {
        const Platform platform{sm_counts[k], Rational(1)};
        const ds_platform pl = detail::platform_of(platform);
        PerM& P = per[k];
        P.st.assign(nv, 0);
        P.bounds.assign(nv * 10, 0);
        ds_results r{P.st.data(), P.bounds.data(), nullptr};
        detail::check(ds_analyze_batch(&b, &pl, DS_M_PROPOSED | DS_M_GREEDY, &r, dev, nullptr, 0));
        if (runs > 0) {
            ds_greedy_cfg cfg{1, int(runs), seed, 0, 0, 0, 1, 1, 1, 1};
            P.gst.assign(nv * runs, 0);
            P.gmk.assign(nv * runs * 2, 0);
            detail::check(ds_simulate_greedy_batch(&b, &pl, &cfg, P.gst.data(), P.gmk.data(), nullptr, dev));
        }
    }
    std::vector<BenchCell> cells;
    for (std::size_t v = 0; v < nv; ++v) {
        for (std::size_t k = 0; k < sm_counts.size(); ++k) {
            const Platform platform{sm_counts[k], Rational(1)};
            PerM& P = per[k];
            BenchCell c;
            c.fixture = vars[v].name;
            c.sm_count = sm_counts[k];
            c.avg_load = vars[v].avg;
            // the schedule of this variant (detail pass; status errors raise
            // in the reference's loop order)
            const ScheduleScheme scheme = schedule(vars[v].task, platform);
            detail::raise(P.st[v], "run_benchmarks: " + c.fixture);
            c.proposed_bound = dag_makespan_bound(scheme);
            c.greedy_bound = bound_at(P.bounds, v, DS_BOUND_GREEDY);
            SimConfig sim;
            sim.platform = platform;
            c.proposed_sim = simulate_scheme(vars[v].task, scheme, sim).makespan;
            double s = 0.0, sq = 0.0, mx = 0.0;
            for (std::size_t r = 0; r < runs; ++r) {
                detail::raise(P.gst[v * runs + r], "run_benchmarks: greedy " + c.fixture);
                const double mk = to_double(Rational(BigInt(P.gmk[2 * (v * runs + r)]),
                                                     BigInt(P.gmk[2 * (v * runs + r) + 1])));
                s += mk;
                sq += mk * mk;
                mx = std::max(mx, mk);
            }
            c.greedy_sim_max = mx;
            c.greedy_sim_avg = s / greedy_runs;
            c.greedy_sim_std = std::sqrt(std::max(0.0, sq / greedy_runs - c.greedy_sim_avg * c.greedy_sim_avg));
            cells.push_back(std::move(c));
        }
    }
    return cells;
}

void write_bench_table(const std::vector<BenchCell>& cells, std::ostream& out) {
    out << "fixture,M,avg_load,proposed_bound,greedy_bound,proposed_sim,greedy_sim_max,greedy_sim_avg,greedy_sim_std\n";
    char buf[128];
    for (const BenchCell& c : cells) {
        std::snprintf(buf, sizeof(buf), "%.4f,%.4f,%.4f", c.greedy_sim_max, c.greedy_sim_avg, c.greedy_sim_std);
        out << c.fixture << "," << c.sm_count << "," << c.avg_load << "," << format_fixed(c.proposed_bound, 4) << ","
            << format_fixed(c.greedy_bound, 4) << "," << format_fixed(c.proposed_sim, 4) << "," << buf << "\n";
    }
}

}  // namespace dagsched

// TEST INFRASTRUCTURE — oracle restatement (see restate.hpp for the map of
// reference lines). Written against the reference's observable semantics,
// with its own data layout: index-ordered arrays and word bitmasks.
#include "restate.hpp"

#include "../../include/dagsched_b200.h"

#include <algorithm>
#include <climits>
#include <cmath>
#include <deque>
#include <random>
#include <set>
#include <sstream>

namespace orc {

namespace {

inline bool bit(const Bits& b, int i) { return (b[i >> 6] >> (i & 63)) & 1; }
inline void setb(Bits& b, int i) { b[i >> 6] |= uint64_t(1) << (i & 63); }

Q qmax(const Q& a, const Q& b) { return a < b ? b : a; }

}  // namespace

// ---------------------------------------------------------- exec_model.cpp
void check_platform(const Platform& p) {  // exec_model.hpp:14-18
    if (p.M < 1) throw std::invalid_argument("sm_count must be >= 1");
    if (p.tmin <= Q(0)) throw std::invalid_argument("t_min must be positive");
}

Q exec_time(const Q& load, long long m, const Platform& p) {  // exec_model.cpp:7-14
    check_platform(p);
    if (m < 1) throw std::invalid_argument("parallelism must be >= 1");
    if (load <= Q(0)) throw std::invalid_argument("load must be positive");
    long long passes = (m + p.M - 1) / p.M;
    Q c = Q(passes) * load / Q(m);
    return c < p.tmin ? p.tmin : c;
}

int max_par(const Q& load, const Platform& p) {  // exec_model.cpp:16-23
    check_platform(p);
    if (load <= Q(0)) throw std::invalid_argument("load must be positive");
    i128 m = q_floor(load / p.tmin);
    if (m < 1) return 1;
    if (m > INT_MAX) return INT_MAX;
    return int(m);
}

// ------------------------------------------------------------------ dag.cpp
Dag make_dag(std::vector<Q> loads, std::vector<std::pair<long long, long long>> edges,
             const Q& min_load) {
    // dag.cpp:25-41: empty, (ids are dense indices: no duplicates), load floor
    if (loads.empty()) throw ValidationError(DS_E_EMPTY, "task has no nodes");
    const int n = int(loads.size());
    for (int i = 0; i < n; ++i) {
        if (loads[i] < min_load) {
            throw ValidationError(DS_E_LOAD, "node " + std::to_string(i) + ": load " +
                                                 q_str(loads[i]) + " below minimum");
        }
    }
    Dag g;
    g.n = n;
    g.load = std::move(loads);
    // dag.cpp:48-67: sorted/deduped edges checked in order
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    g.pred.assign(n, {});
    g.succ.assign(n, {});
    for (auto [u, v] : edges) {
        if (u < 0 || v < 0 || u >= n || v >= n) {
            throw ValidationError(DS_E_EDGE, "edge references unknown node");
        }
        if (u == v) throw ValidationError(DS_E_SELFLOOP, "cycle detected: self-loop");
        g.succ[u].push_back(int(v));
        g.pred[v].push_back(int(u));
        g.edges.emplace_back(int(u), int(v));
    }
    // dag.cpp:69-95: Kahn (FIFO, index-ordered seeds) doubles as cycle check
    std::vector<int> indeg(n);
    std::vector<int> fifo;
    for (int i = 0; i < n; ++i) {
        indeg[i] = int(g.pred[i].size());
        if (!indeg[i]) fifo.push_back(i);
    }
    for (size_t h = 0; h < fifo.size(); ++h) {
        for (int v : g.succ[fifo[h]]) {
            if (--indeg[v] == 0) fifo.push_back(v);
        }
    }
    if (int(fifo.size()) != n) throw ValidationError(DS_E_CYCLE, "cycle detected involving nodes");
    g.topo = fifo;
    // dag.cpp:97-110: single source, single sink
    int ns = 0, nk = 0;
    for (int i = 0; i < n; ++i) {
        ns += g.pred[i].empty();
        nk += g.succ[i].empty();
    }
    if (ns != 1) throw ValidationError(DS_E_SOURCES, "expected a single source node");
    if (nk != 1) throw ValidationError(DS_E_SINKS, "expected a single sink node");
    // dag.cpp:112-124: closures in topological / reverse order
    const int w = g.words();
    g.anc.assign(n, Bits(w, 0));
    g.desc.assign(n, Bits(w, 0));
    for (int u : g.topo) {
        for (int p : g.pred[u]) {
            for (int k = 0; k < w; ++k) g.anc[u][k] |= g.anc[p][k];
            setb(g.anc[u], p);
        }
    }
    for (auto it = g.topo.rbegin(); it != g.topo.rend(); ++it) {
        for (int s : g.succ[*it]) {
            for (int k = 0; k < w; ++k) g.desc[*it][k] |= g.desc[s][k];
            setb(g.desc[*it], s);
        }
    }
    // dag.cpp:126-135: W^anc = own load + ancestors' loads
    g.wanc.resize(n);
    for (int i = 0; i < n; ++i) {
        Q s = g.load[i];
        for (int j = 0; j < n; ++j) {
            if (bit(g.anc[i], j)) s = s + g.load[j];
        }
        g.wanc[i] = s;
    }
    return g;
}

std::vector<int> join_nodes(const Dag& g) {  // dag.cpp:218-230 (ascending W^anc, ties id)
    std::vector<int> j;
    for (int i = 0; i < g.n; ++i) {
        if (g.pred[i].size() >= 2) j.push_back(i);
    }
    std::sort(j.begin(), j.end(), [&](int a, int b) {
        if (g.wanc[a] != g.wanc[b]) return g.wanc[a] < g.wanc[b];
        return a < b;
    });
    return j;
}

// ------------------------------------------------------------- division.cpp
std::vector<std::vector<int>> build_blocks(const Dag& g, std::vector<int>* residual_flag) {
    // division.cpp:10-30: per join (in join order) the unassigned ancestors,
    // then the residual block (always emitted, possibly empty).
    std::vector<std::vector<int>> out;
    std::vector<char> taken(g.n, 0);
    for (int j : join_nodes(g)) {
        std::vector<int> b;
        for (int i = 0; i < g.n; ++i) {
            if (bit(g.anc[j], i) && !taken[i]) {
                b.push_back(i);
                taken[i] = 1;
            }
        }
        out.push_back(b);
        if (residual_flag) residual_flag->push_back(0);
    }
    std::vector<int> rest;
    for (int i = 0; i < g.n; ++i) {
        if (!taken[i]) rest.push_back(i);
    }
    out.push_back(rest);
    if (residual_flag) residual_flag->push_back(1);
    return out;
}

std::vector<std::vector<int>> local_paths(const Dag& g, const std::vector<int>& block) {
    // division.cpp:32-65. With NDEBUG (the reference's Release build) the
    // "unique in-block predecessor" assert is compiled out and the last
    // (largest-id) in-block predecessor wins; kept literally.
    std::vector<char> in(g.n, 0);
    for (int v : block) in[v] = 1;
    std::vector<std::vector<int>> paths;
    for (int v : block) {
        bool sink = true;
        for (int s : g.succ[v]) {
            if (in[s]) {
                sink = false;
                break;
            }
        }
        if (!sink) continue;
        std::vector<int> rev{v};
        int cur = v;
        for (;;) {
            int lp = -1;
            for (int p : g.pred[cur]) {
                if (in[p]) lp = p;
            }
            if (lp < 0) break;
            rev.push_back(lp);
            cur = lp;
        }
        paths.emplace_back(rev.rbegin(), rev.rend());
    }
    return paths;
}

std::vector<std::vector<int>> build_groups(const Dag& g, const Platform& p) {
    // division.cpp:67-126
    check_platform(p);
    std::vector<std::vector<int>> groups;
    for (const auto& block : build_blocks(g)) {
        if (block.empty()) continue;
        std::vector<std::deque<int>> paths;
        for (auto& pth : local_paths(g, block)) paths.emplace_back(pth.begin(), pth.end());
        while (!paths.empty()) {
            std::vector<int> heads;
            for (auto& pth : paths) {
                if (std::find(heads.begin(), heads.end(), pth.front()) == heads.end()) {
                    heads.push_back(pth.front());
                }
            }
            std::sort(heads.begin(), heads.end(), [&](int a, int b) {
                if (g.wanc[a] != g.wanc[b]) return g.wanc[a] > g.wanc[b];
                return a < b;
            });
            if (int(heads.size()) > p.M) heads.resize(p.M);
            bool big = false;
            for (int v : heads) big |= max_par(g.load[v], p) >= p.M;
            if (big) {
                int pick = heads.front(), best = 0;
                for (int v : heads) {
                    int mp = max_par(g.load[v], p);
                    if (mp > best || (mp == best && v < pick)) {
                        best = mp;
                        pick = v;
                    }
                }
                heads.assign(1, pick);
            }
            for (auto& pth : paths) {
                if (std::find(heads.begin(), heads.end(), pth.front()) != heads.end()) {
                    pth.pop_front();
                }
            }
            paths.erase(std::remove_if(paths.begin(), paths.end(),
                                       [](const std::deque<int>& d) { return d.empty(); }),
                        paths.end());
            std::sort(heads.begin(), heads.end());
            groups.push_back(heads);
        }
    }
    return groups;
}

// ------------------------------------------------------------ scheduler.cpp
bool operator<(const Ent& a, const Ent& b) {  // scheduler.hpp:19-27 (field order)
    if (a.origin != b.origin) return a.origin < b.origin;
    if (a.gen != b.gen) return a.gen < b.gen;
    return a.part < b.part;
}
bool operator==(const Ent& a, const Ent& b) {
    return a.origin == b.origin && a.gen == b.gen && a.part == b.part;
}
std::string ent_str(const Ent& e) {  // scheduler.cpp:9-17
    std::string s = std::to_string(e.origin);
    if (e.part == 1) s += ":p" + std::to_string(e.gen);
    if (e.part == 2) s += ":r" + std::to_string(e.gen);
    return s;
}

std::vector<int> apportion(const std::vector<Q>& loads, const std::vector<int>& caps,
                           const Platform& p) {
    // scheduler.cpp:35-95: floor quotas clamped to [1, cap]; shed to the
    // cheapest slowdown (first strict min); fill to the largest current
    // exec, ties larger remainder, then first index.
    const int k = int(loads.size());
    Q W(0);
    for (const Q& l : loads) W = W + l;
    std::vector<Q> quota(k), rem(k);
    std::vector<int> m(k);
    long long total = 0;
    for (int i = 0; i < k; ++i) {
        quota[i] = loads[i] * Q(p.M) / W;
        i128 f = q_floor(quota[i]);
        long long b = std::max<long long>(1, std::min<long long>((long long)f, caps[i]));
        m[i] = int(b);
        total += b;
        rem[i] = quota[i] - Q(f, 1);
    }
    while (total > p.M) {
        int pick = -1;
        Q best;
        for (int i = 0; i < k; ++i) {
            if (m[i] <= 1) continue;
            Q slowed = exec_time(loads[i], m[i] - 1, p);
            if (pick < 0 || slowed < best) {
                pick = i;
                best = slowed;
            }
        }
        --m[pick];
        --total;
    }
    long long capsum = 0;
    for (int c : caps) capsum += c;
    const long long target = std::min<long long>(p.M, capsum);
    while (total < target) {
        int pick = -1;
        Q be, br;
        for (int i = 0; i < k; ++i) {
            if (m[i] >= caps[i]) continue;
            Q cur = exec_time(loads[i], m[i], p);
            if (pick < 0 || cur > be || (cur == be && rem[i] > br)) {
                pick = i;
                be = cur;
                br = rem[i];
            }
        }
        ++m[pick];
        ++total;
    }
    return m;
}

namespace {
struct EP {
    Ent e;
    bool extra;
};
struct Pend {
    bool live = true;
    Ent id;
    Q load;
    std::vector<EP> eps;
};
struct Draft {
    Ent e;
    Q load;
    int m;
    Q exec;
    int group;
    bool launched;
    int origin;
    std::vector<EP> eps;
};
}  // namespace

Scheme schedule(const Dag& g, const Platform& p) {
    // scheduler.cpp:175-427
    check_platform(p);
    for (int i = 0; i < g.n; ++i) {
        if (g.load[i] < p.tmin) {
            throw ValidationError(DS_E_LOAD_TMIN, "load below the platform time unit");
        }
    }
    const int M = p.M;
    const auto division = build_groups(g, p);
    const int n = g.n, w = g.words();
    std::vector<Pend> pend(n);
    for (int i = 0; i < n; ++i) pend[i] = Pend{true, Ent{i, 0, 0}, g.load[i], {}};
    std::vector<Draft> drafts;
    std::vector<int> done(n, -1), gen(n, 0);
    std::vector<std::vector<Ent>> chain(n);
    Scheme s;
    s.plat = p;

    auto recorded_group = [&](const Ent& e) {
        for (const Draft& d : drafts) {
            if (d.e == e) return d.group;
        }
        return -1;
    };
    auto released = [&](int c, int gidx) {  // scheduler.cpp:202-212
        for (int o : g.pred[c]) {
            if (done[o] < 0 || done[o] >= gidx) return false;
        }
        for (const EP& d : pend[c].eps) {
            int rg = recorded_group(d.e);
            if (rg < 0 || rg >= gidx) return false;
        }
        return true;
    };

    for (const auto& grp : division) {
        std::vector<int> org;
        for (int v : grp) {
            if (pend[v].live) org.push_back(v);
        }
        if (org.empty()) continue;
        const int gidx = int(s.groups.size());
        std::vector<Q> loads;
        std::vector<int> caps;
        for (int v : org) {
            loads.push_back(pend[v].load);
            caps.push_back(std::min(max_par(pend[v].load, p), M));
        }
        std::vector<int> m = apportion(loads, caps, p);

        Group plan;
        plan.index = gidx;
        int used = 0;
        for (size_t i = 0; i < org.size(); ++i) {
            const Pend& pd = pend[org[i]];
            plan.members.push_back(Member{pd.id, pd.load, m[i], exec_time(pd.load, m[i], p)});
            used += m[i];
        }
        plan.resp = plan.members[0].exec;
        plan.bottleneck = plan.members[0].e;
        for (const Member& mb : plan.members) {
            if (mb.exec > plan.resp) {
                plan.resp = mb.exec;
                plan.bottleneck = mb.e;
            }
        }
        plan.spare = M - used;
        plan.spare_cap = plan.resp * Q(plan.spare);

        // candidate pool: concurrent sets of pending members minus the whole
        // division group (scheduler.cpp:253-258)
        Bits ingrp(w, 0), pool(w, 0);
        for (int v : grp) setb(ingrp, v);
        for (int v : org) {
            for (int c = 0; c < n; ++c) {
                if (c == v || bit(g.anc[v], c) || bit(g.desc[v], c) || bit(ingrp, c)) continue;
                setb(pool, c);
            }
        }
        std::vector<int> cands;
        for (int c = 0; c < n; ++c) {  // scheduler.cpp:260-274
            if (!bit(pool, c)) continue;
            bool src = true;
            for (int q : g.pred[c]) src &= !bit(pool, q);
            if (!src) continue;
            if (pend[c].live && released(c, gidx)) cands.push_back(c);
        }
        std::sort(cands.begin(), cands.end(), [&](int a, int b) {
            if (g.wanc[a] != g.wanc[b]) return g.wanc[a] > g.wanc[b];
            return a < b;
        });

        int spare = plan.spare;
        std::vector<char> whole(n, 0);
        std::vector<Ent> launched;
        for (int c : cands) {  // scheduler.cpp:286-330
            if (spare < 1) break;
            Pend& cd = pend[c];
            int mc = std::min(max_par(cd.load, p), spare);
            Q dur = exec_time(cd.load, mc, p);
            if (dur <= plan.resp) {
                drafts.push_back(Draft{cd.id, cd.load, mc, dur, gidx, true, c, cd.eps});
                chain[c].push_back(cd.id);
                plan.launches.push_back(Launch{cd.id, mc, dur});
                launched.push_back(cd.id);
                whole[c] = 1;
                done[c] = gidx;
                cd.live = false;
                spare -= mc;
            } else {
                int gn = ++gen[c];
                Ent par{c, gn, 1}, res{c, gn, 2};
                Q pl = Q(mc) * plan.resp;
                Q rl = cd.load - pl;
                drafts.push_back(Draft{par, pl, mc, plan.resp, gidx, true, c, cd.eps});
                chain[c].push_back(par);
                plan.launches.push_back(Launch{par, mc, plan.resp});
                launched.push_back(par);
                std::vector<EP> eps = cd.eps;
                eps.push_back(EP{par, false});
                cd = Pend{true, res, rl, eps};
                // scheduler.cpp:318-328: `cand` is a reference into `pending`
                // and is reassigned to the residual before the record is
                // built, so the reference's SegmentationRecord::source is the
                // residual id, not the entity that was split. Kept for parity.
                s.segs.push_back(Seg{cd.id, par, res, pl, rl, gidx});
                spare -= mc;
                break;
            }
        }
        // extra dependencies (scheduler.cpp:336-346)
        for (const Ent& e : launched) {
            for (int sc : g.succ[plan.bottleneck.origin]) pend[sc].eps.push_back(EP{e, true});
        }
        for (int c : cands) {
            if (!whole[c]) pend[c].eps.push_back(EP{plan.bottleneck, true});
        }
        for (size_t i = 0; i < org.size(); ++i) {  // commit (scheduler.cpp:348-356)
            int v = org[i];
            drafts.push_back(Draft{pend[v].id, pend[v].load, m[i], plan.members[i].exec, gidx,
                                   false, v, pend[v].eps});
            chain[v].push_back(pend[v].id);
            done[v] = gidx;
            pend[v].live = false;
        }
        s.groups.push_back(plan);
    }
    for (int i = 0; i < n; ++i) {
        if (pend[i].live) throw std::logic_error("scheduling finished with unplaced kernels");
    }

    // materialise (scheduler.cpp:365-385)
    std::sort(drafts.begin(), drafts.end(), [](const Draft& a, const Draft& b) { return a.e < b.e; });
    std::set<std::pair<Ent, Ent>> extra;
    for (const Draft& d : drafts) {
        std::set<Ent> preds;
        for (int o : g.pred[d.origin]) preds.insert(chain[o].back());
        for (const EP& ep : d.eps) {
            preds.insert(ep.e);
            if (ep.extra) extra.insert({ep.e, d.e});
        }
        s.ents.push_back(Record{d.e, d.load, d.m, d.exec, d.group, d.launched,
                                std::vector<Ent>(preds.begin(), preds.end())});
    }
    s.extra.assign(extra.begin(), extra.end());

    // self-checks (scheduler.cpp:389-424)
    {
        const size_t E = s.ents.size();
        auto idx = [&](const Ent& e) {
            auto it = std::lower_bound(s.ents.begin(), s.ents.end(), e,
                                       [](const Record& r, const Ent& v) { return r.e < v; });
            return size_t(it - s.ents.begin());
        };
        std::vector<size_t> indeg(E, 0);
        std::vector<std::vector<size_t>> out(E);
        for (size_t i = 0; i < E; ++i) {
            for (const Ent& pe : s.ents[i].preds) {
                out[idx(pe)].push_back(i);
                ++indeg[i];
            }
        }
        std::vector<size_t> q;
        for (size_t i = 0; i < E; ++i) {
            if (!indeg[i]) q.push_back(i);
        }
        for (size_t h = 0; h < q.size(); ++h) {
            for (size_t v : out[q[h]]) {
                if (--indeg[v] == 0) q.push_back(v);
            }
        }
        if (q.size() != E) throw std::logic_error("augmented dependency graph has a cycle");
    }
    for (const Group& gp : s.groups) {
        int t = 0;
        for (const Member& mb : gp.members) t += mb.m;
        for (const Launch& l : gp.launches) t += l.m;
        if (t > M) throw std::logic_error("group allocation exceeds the device");
    }
    return s;
}

// ------------------------------------------------------------- analysis.cpp
namespace {
Q longest_path(const Dag& g, const std::vector<Q>& wgt) {  // analysis.cpp:11-24
    std::vector<Q> best(g.n);
    Q result(0);
    for (int v : g.topo) {
        Q in(0);
        for (int pp : g.pred[v]) in = qmax(in, best[pp]);
        best[v] = in + wgt[v];
        result = qmax(result, best[v]);
    }
    return result;
}
}  // namespace

Q proposed_bound(const Scheme& s) {  // analysis.cpp:34-38
    Q t(0);
    for (const Group& gp : s.groups) t = t + gp.resp;
    return t;
}
Q greedy_bound(const Dag& g, const Platform& p) {  // analysis.cpp:40-48
    check_platform(p);
    Q t(0);
    for (int i = 0; i < g.n; ++i) {
        t = t + exec_time(g.load[i], std::min(max_par(g.load[i], p), p.M), p);
    }
    return t;
}
Q greedy_unaware_bound(const Dag& g, const Platform& p) {  // analysis.cpp:50-57
    check_platform(p);
    Q t(0);
    for (int i = 0; i < g.n; ++i) t = t + exec_time(g.load[i], max_par(g.load[i], p), p);
    return t;
}
Q graham_para_bound(const Dag& g, const Platform& p) {  // analysis.cpp:59-70
    check_platform(p);
    Q work(0);
    for (int i = 0; i < g.n; ++i) work = work + Q(q_ceil(g.load[i] / p.tmin), 1) * p.tmin;
    Q chain = longest_path(g, std::vector<Q>(g.n, p.tmin));
    return chain + (work - chain) / Q(p.M);
}
Q lower_bound(const Dag& g, const Platform& p) {  // analysis.cpp:72-81
    check_platform(p);
    Q total(0);
    for (int i = 0; i < g.n; ++i) total = total + g.load[i];
    std::vector<Q> wgt(g.n);
    for (int i = 0; i < g.n; ++i) {
        wgt[i] = exec_time(g.load[i], std::min(max_par(g.load[i], p), p.M), p);
    }
    return qmax(total / Q(p.M), longest_path(g, wgt));
}

// ------------------------------------------------------------ generator.cpp
Dag generate(const GenCfg& c) {
    // generator.cpp:9-22 (config check)
    if (c.depth_min < 2 || c.depth_max < c.depth_min) throw std::invalid_argument("depth range");
    if (c.max_width < 2) throw std::invalid_argument("max_width must be >= 2");
    if (c.tmin <= Q(0)) throw std::invalid_argument("t_min must be positive");
    if (c.avg_load < c.tmin) throw std::invalid_argument("avg_load must be >= t_min");
    if (c.jitter < 0 || c.jitter > 1) throw std::invalid_argument("load_jitter");
    if (c.density < 0 || c.density > 1) throw std::invalid_argument("edge_density");
    // generator.cpp:24-96 — the RNG call order is the contract:
    // depth; widths; per node (layer order) parent then coins over earlier
    // layers skipping the parent; loads in id order.
    std::mt19937_64 rng(c.seed);
    const int depth = std::uniform_int_distribution<int>(c.depth_min, c.depth_max)(rng);
    std::vector<int> lay_begin{0}, lay_size{1};
    int next = 1;
    for (int l = 0; l < depth - 2; ++l) {
        int wd = std::uniform_int_distribution<int>(2, c.max_width)(rng);
        lay_begin.push_back(next);
        lay_size.push_back(wd);
        next += wd;
    }
    const int sink = next++;
    std::vector<std::pair<long long, long long>> edges;
    std::uniform_real_distribution<double> coin(0.0, 1.0);
    for (size_t l = 1; l < lay_begin.size(); ++l) {
        for (int v = lay_begin[l]; v < lay_begin[l] + lay_size[l]; ++v) {
            size_t pick = std::uniform_int_distribution<std::size_t>(0, lay_size[l - 1] - 1)(rng);
            int parent = lay_begin[l - 1] + int(pick);
            edges.emplace_back(parent, v);
            for (size_t e = 0; e < l; ++e) {
                for (int u = lay_begin[e]; u < lay_begin[e] + lay_size[e]; ++u) {
                    if (u == parent) continue;
                    if (coin(rng) < c.density) edges.emplace_back(u, v);
                }
            }
        }
    }
    std::vector<char> has_child(next, 0);
    for (auto& e : edges) has_child[e.first] = 1;
    for (int v = 0; v < sink; ++v) {
        if (!has_child[v]) edges.emplace_back(v, sink);
    }
    const double avg = q_double(c.avg_load);
    std::uniform_real_distribution<double> ld(avg * (1.0 - c.jitter), avg * (1.0 + c.jitter));
    std::vector<Q> loads;
    for (int v = 0; v < next; ++v) {
        double x = ld(rng);
        Q l = c.integer_loads ? Q(std::llround(x / q_double(c.tmin))) * c.tmin
                              : Q::of(std::llround(x * 1000.0), 1000);
        if (l < c.tmin) l = c.tmin;
        loads.push_back(l);
    }
    if (c.exact_mean) {
        Q sum(0);
        for (const Q& l : loads) sum = sum + l;
        Q f = c.avg_load * Q((long long)loads.size()) / sum;
        for (Q& l : loads) {
            l = l * f;
            if (l < c.tmin) l = c.tmin;
        }
    }
    return make_dag(std::move(loads), std::move(edges), c.tmin);
}

// ---------------------------------------------------- task_io.cpp:94-148
std::string scheme_json(const Scheme& s) {
    std::ostringstream o;
    auto qs = [](const Q& q) { return "\"" + q_str(q) + "\""; };
    auto es = [](const Ent& e) { return "\"" + ent_str(e) + "\""; };
    o << "{\"platform\": {\"sm_count\": " << s.plat.M << ", \"t_min\": " << qs(s.plat.tmin)
      << "}, \"groups\": [";
    for (size_t i = 0; i < s.groups.size(); ++i) {
        const Group& g = s.groups[i];
        o << (i ? ", " : "") << "{\"index\": " << g.index << ", \"members\": [";
        for (size_t k = 0; k < g.members.size(); ++k) {
            const Member& m = g.members[k];
            o << (k ? ", " : "") << "{\"entity\": " << es(m.e) << ", \"load\": " << qs(m.load)
              << ", \"parallelism\": " << m.m << ", \"exec_time\": " << qs(m.exec) << "}";
        }
        o << "], \"spare_sms\": " << g.spare << ", \"spare_capacity\": " << qs(g.spare_cap)
          << ", \"response\": " << qs(g.resp) << ", \"bottleneck\": " << es(g.bottleneck)
          << ", \"launches\": [";
        for (size_t k = 0; k < g.launches.size(); ++k) {
            const Launch& l = g.launches[k];
            o << (k ? ", " : "") << "{\"entity\": " << es(l.e) << ", \"parallelism\": " << l.m
              << ", \"duration\": " << qs(l.dur) << "}";
        }
        o << "]}";
    }
    o << "], \"segmentations\": [";
    for (size_t i = 0; i < s.segs.size(); ++i) {
        const Seg& g = s.segs[i];
        o << (i ? ", " : "") << "{\"source\": " << es(g.src) << ", \"parallel\": " << es(g.par)
          << ", \"residual\": " << es(g.res) << ", \"parallel_load\": " << qs(g.par_load)
          << ", \"residual_load\": " << qs(g.res_load) << ", \"group\": " << g.group << "}";
    }
    o << "], \"extra_deps\": [";
    for (size_t i = 0; i < s.extra.size(); ++i) {
        o << (i ? ", " : "") << "[" << es(s.extra[i].first) << ", " << es(s.extra[i].second) << "]";
    }
    o << "], \"entities\": [";
    for (size_t i = 0; i < s.ents.size(); ++i) {
        const Record& r = s.ents[i];
        o << (i ? ", " : "") << "{\"id\": " << es(r.e) << ", \"load\": " << qs(r.load)
          << ", \"parallelism\": " << r.m << ", \"exec_time\": " << qs(r.exec)
          << ", \"group\": " << r.group << ", \"launched\": " << (r.launched ? "true" : "false")
          << ", \"preds\": [";
        for (size_t k = 0; k < r.preds.size(); ++k) o << (k ? ", " : "") << es(r.preds[k]);
        o << "]}";
    }
    o << "]}";
    return o.str();
}

}  // namespace orc

// Kept C++ API — Alg. 2. schedule()/schedule_batch() run on the device
// (ds_schedule_batch: K1 in detail mode) and only the bookkeeping the
// reference does after the fact (scheduler.cpp:361-385: origin predecessors
// resolved to the last segment of the origin's chain, entity predecessors,
// extra-dependency set) is replayed here from the device's records.
// scale_parallelism / parallel_candidates are the reference's standalone
// per-group helpers (scheduler.cpp:99-146), answered on the host.
#include "dagsched/scheduler.hpp"

#include "device.hpp"

#include <algorithm>
#include <map>
#include <stdexcept>

namespace dagsched {

std::string to_string(const EntityId& id) {
    const std::string o = std::to_string(id.origin);
    switch (id.part) {
        case EntityId::Part::parallel: return o + ":p" + std::to_string(id.generation);
        case EntityId::Part::residual: return o + ":r" + std::to_string(id.generation);
        default: return o;
    }
}

const EntityRecord& ScheduleScheme::entity(const EntityId& id) const {
    auto it = std::lower_bound(entities.begin(), entities.end(), id,
                               [](const EntityRecord& r, const EntityId& v) { return r.id < v; });
    if (it == entities.end() || it->id != id) throw std::out_of_range("unknown entity " + to_string(id));
    return *it;
}

namespace {

// apportion (scheduler.cpp:35-95): floor quotas clamped to [1, cap], shed to
// the smallest slowdown, fill to the largest current exec (ties: larger
// remainder, then first index)
std::vector<int> apportion(const std::vector<Rational>& loads, const std::vector<int>& caps, const Platform& p) {
    const std::size_t k = loads.size();
    Rational W;
    for (const Rational& l : loads) W += l;
    std::vector<Rational> q(k), rem(k);
    std::vector<int> m(k);
    long long tot = 0;
    for (std::size_t i = 0; i < k; ++i) {
        q[i] = loads[i] * Rational(p.sm_count, 1) / W;
        const BigInt f = floor_to_int(q[i]);
        m[i] = int(std::max(1LL, std::min<long long>(to_int64(f), caps[i])));
        rem[i] = q[i] - Rational(f, 1);
        tot += m[i];
    }
    while (tot > p.sm_count) {
        std::size_t pick = k;
        Rational best;
        for (std::size_t i = 0; i < k; ++i) {
            if (m[i] <= 1) continue;
            const Rational s = exec_time(loads[i], m[i] - 1, p);
            if (pick == k || s < best) pick = i, best = s;
        }
        if (pick == k) throw std::logic_error("apportion: cannot shed");
        --m[pick], --tot;
    }
    long long capsum = 0;
    for (int c : caps) capsum += c;
    while (tot < std::min<long long>(p.sm_count, capsum)) {
        std::size_t pick = k;
        Rational be, br;
        for (std::size_t i = 0; i < k; ++i) {
            if (m[i] >= caps[i]) continue;
            const Rational cur = exec_time(loads[i], m[i], p);
            if (pick == k || cur > be || (cur == be && rem[i] > br)) pick = i, be = cur, br = rem[i];
        }
        if (pick == k) throw std::logic_error("apportion: cannot fill");
        ++m[pick], ++tot;
    }
    return m;
}

Rational rat(int64_t n, int64_t d) { return Rational(BigInt(n), BigInt(d)); }

EntityId eid(const DagTask& t, const ds_entity_rec& r) {
    return EntityId{t.nodes()[r.origin].id, r.generation, EntityId::Part(r.part)};
}

// The reference's closing self-checks (scheduler.cpp:389-424): the augmented
// graph is acyclic (Kahn over the entity preds) and no group holds more than
// M SMs; either failure is a scheduler bug -> std::logic_error, as there.
void verify(const ScheduleScheme& s, int M) {
    std::map<EntityId, std::size_t> idx;
    for (std::size_t i = 0; i < s.entities.size(); ++i) idx[s.entities[i].id] = i;
    std::vector<std::size_t> indeg(s.entities.size(), 0), queue;
    std::vector<std::vector<std::size_t>> succ(s.entities.size());
    for (std::size_t i = 0; i < s.entities.size(); ++i) {
        for (const EntityId& p : s.entities[i].preds) {
            auto it = idx.find(p);
            if (it == idx.end()) throw std::logic_error("entity predecessor is not an entity");
            succ[it->second].push_back(i);
            ++indeg[i];
        }
    }
    for (std::size_t i = 0; i < indeg.size(); ++i)
        if (indeg[i] == 0) queue.push_back(i);
    for (std::size_t h = 0; h < queue.size(); ++h)
        for (std::size_t v : succ[queue[h]])
            if (--indeg[v] == 0) queue.push_back(v);
    if (queue.size() != s.entities.size()) throw std::logic_error("augmented dependency graph has a cycle");
    for (const GroupPlan& g : s.groups) {
        long long total = 0;
        for (const MemberPlan& mp : g.members) total += mp.parallelism;
        for (const LaunchRecord& l : g.launches) total += l.parallelism;
        if (total > M) throw std::logic_error("group allocation exceeds the device");
    }
}

ScheduleScheme materialise(const DagTask& t, const Platform& plat, const ds_entity_rec* er, int ne,
                           const ds_group_rec* gr, int ng, const std::uint64_t* unl) {
    ScheduleScheme s;
    s.platform = plat;
    const std::size_t n = t.size();
    struct Dep {
        EntityId e;
        bool extra;
    };
    std::vector<std::vector<Dep>> pending(n);             // entity preds per pending node
    std::vector<std::vector<EntityId>> chain(n);           // entities per origin, in order
    std::vector<std::vector<Dep>> rec(ne);                 // entity preds frozen at record time
    std::vector<std::vector<std::uint32_t>> succ(n);
    for (std::uint32_t w : t.edge_words()) succ[w >> 16].push_back(w & 0xffff);
    for (int g = 0; g < ng; ++g) {
        const ds_group_rec& G = gr[g];
        GroupPlan plan;
        plan.index = std::size_t(g);
        plan.spare_sms = G.spare_sms;
        plan.response = rat(G.resp_num, G.resp_den);
        plan.spare_capacity = plan.response * Rational(G.spare_sms, 1);
        plan.bottleneck = eid(t, er[G.bottleneck]);
        const int L0 = G.first_entity, L1 = L0 + G.n_launches, M1 = L1 + G.n_members;
        for (int i = L0; i < L1; ++i) {  // launches, in launch order
            const ds_entity_rec& r = er[i];
            rec[i] = pending[r.origin];
            chain[r.origin].push_back(eid(t, r));
            plan.launches.push_back(LaunchRecord{eid(t, r), r.parallelism, rat(r.exec_num, r.exec_den)});
            if (r.part == 1) {  // a split: the residual inherits + waits for its parallel segment
                const EntityId res{t.nodes()[r.origin].id, r.generation, EntityId::Part::residual};
                // SegmentationRecord::source aliases the residual (scheduler.cpp:318-328)
                s.segmentations.push_back(SegmentationRecord{res, eid(t, r), res, rat(r.load_num, r.load_den),
                                                             rat(r.res_num, r.res_den), std::size_t(g)});
                pending[r.origin].push_back(Dep{eid(t, r), false});
            }
        }
        for (int i = L0; i < L1; ++i)  // launched -> successors of the bottleneck
            for (std::uint32_t sc : succ[er[G.bottleneck].origin]) pending[sc].push_back(Dep{eid(t, er[i]), true});
        const std::uint64_t* unl_g = unl + std::size_t(g) * ((n + 63) / 64);
        for (std::size_t c = 0; c < n; ++c)  // bottleneck -> unlaunched candidates
            if ((unl_g[c >> 6] >> (c & 63)) & 1) pending[c].push_back(Dep{plan.bottleneck, true});
        for (int i = L1; i < M1; ++i) {
            const ds_entity_rec& r = er[i];
            rec[i] = pending[r.origin];
            chain[r.origin].push_back(eid(t, r));
            plan.members.push_back(
                MemberPlan{eid(t, r), rat(r.load_num, r.load_den), r.parallelism, rat(r.exec_num, r.exec_den)});
        }
        s.groups.push_back(std::move(plan));
    }
    std::set<std::pair<EntityId, EntityId>> extra;
    for (int i = 0; i < ne; ++i) {
        const ds_entity_rec& r = er[i];
        EntityRecord e;
        e.id = eid(t, r);
        e.load = rat(r.load_num, r.load_den);
        e.parallelism = r.parallelism;
        e.exec = rat(r.exec_num, r.exec_den);
        e.group = r.group;
        e.launched = r.launched != 0;
        std::set<EntityId> preds;
        for (NodeId o : t.predecessors(e.id.origin)) preds.insert(chain[t.index_of(o)].back());
        for (const Dep& d : rec[i]) {
            preds.insert(d.e);
            if (d.extra) extra.insert({d.e, e.id});
        }
        e.preds.assign(preds.begin(), preds.end());
        s.entities.push_back(std::move(e));
    }
    std::sort(s.entities.begin(), s.entities.end(), [](const EntityRecord& a, const EntityRecord& b) {
        return a.id < b.id;
    });
    s.extra_deps.assign(extra.begin(), extra.end());
    verify(s, plat.sm_count);
    return s;
}

}  // namespace

std::map<NodeId, int> scale_parallelism(const std::vector<NodeId>& group, const DagTask& task,
                                        const Platform& platform) {
    platform.check();
    std::vector<NodeId> ids = group;
    std::sort(ids.begin(), ids.end());
    std::vector<Rational> loads;
    std::vector<int> caps;
    for (NodeId v : ids) {
        loads.push_back(task.load(v));
        caps.push_back(std::min(max_parallelism(task.load(v), platform), platform.sm_count));
    }
    const std::vector<int> m = apportion(loads, caps, platform);
    std::map<NodeId, int> out;
    for (std::size_t i = 0; i < ids.size(); ++i) out[ids[i]] = m[i];
    return out;
}

std::vector<NodeId> parallel_candidates(const std::vector<NodeId>& group, const DagTask& task,
                                        const std::set<NodeId>& released) {
    const std::set<NodeId> in(group.begin(), group.end());
    std::set<NodeId> pool;
    for (NodeId v : group)
        for (NodeId c : task.concurrent_set(v))
            if (!in.count(c)) pool.insert(c);
    std::vector<NodeId> out;
    for (NodeId c : pool) {
        const auto pr = task.predecessors(c);
        const bool src = std::none_of(pr.begin(), pr.end(), [&](NodeId p) { return pool.count(p) > 0; });
        if (src && released.count(c)) out.push_back(c);
    }
    std::sort(out.begin(), out.end(), [&](NodeId a, NodeId b) {
        const Rational wa = task.cumulative_ancestor_workload(a), wb = task.cumulative_ancestor_workload(b);
        return wa != wb ? wa > wb : a < b;
    });
    return out;
}

namespace detail {
std::vector<ScheduleScheme> schedule_ptrs(const std::vector<const DagTask*>& tasks, const Platform& platform,
                                          int device, std::vector<int64_t>* bounds) {
    const detail::Packed p = detail::pack(tasks);
    const ds_dag_batch b = p.view();
    const ds_platform pl = detail::platform_of(platform);
    const std::size_t nd = tasks.size(), N = p.n_nodes;
    std::vector<int32_t> st(nd);
    std::vector<uint16_t> ne(nd), ng(nd), ndv(nd);
    std::vector<ds_entity_rec> ents(std::max<std::size_t>(2 * N, 1));
    std::vector<ds_group_rec> grps(std::max<std::size_t>(N, 1));
    // unlaunched-candidate masks: n * ceil(n / 64) words per DAG (header layout)
    std::vector<std::size_t> ubase(nd + 1, 0);
    for (std::size_t d = 0; d < nd; ++d) {
        const std::size_t k = tasks[d]->size();
        ubase[d + 1] = ubase[d] + k * ((k + 63) / 64);
    }
    std::vector<std::uint64_t> unl(std::max<std::size_t>(ubase[nd], 1));
    if (bounds) bounds->assign(nd * 10, 0);
    ds_scheme_out out{st.data(), ne.data(), ng.data(), ndv.data(), nullptr, nullptr, ents.data(), grps.data(),
                      bounds ? bounds->data() : nullptr, unl.data()};
    detail::check(ds_schedule_batch(&b, &pl, &out, device));
    std::vector<ScheduleScheme> res;
    res.reserve(nd);
    for (std::size_t d = 0; d < nd; ++d) {
        detail::raise(st[d], "schedule: task " + std::to_string(d));
        const std::size_t n0 = p.node_off[d];
        res.push_back(
            materialise(*tasks[d], platform, ents.data() + 2 * n0, ne[d], grps.data() + n0, ng[d], unl.data() + ubase[d]));
    }
    return res;
}
}  // namespace detail

std::vector<ScheduleScheme> schedule_batch(const std::vector<DagTask>& tasks, const Platform& platform, int device) {
    std::vector<const DagTask*> ptrs;
    for (const DagTask& t : tasks) ptrs.push_back(&t);
    return detail::schedule_ptrs(ptrs, platform, device, nullptr);
}

ScheduleScheme schedule(const DagTask& task, const Platform& platform) {
    return std::move(detail::schedule_ptrs({&task}, platform, detail::devices().front(), nullptr).front());
}

}  // namespace dagsched

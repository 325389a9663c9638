"""Executor (K3) + node workloads (K2) from Python: plans, runs, trace checks.

A plan is what the reference's simulate_scheme (simulator.cpp:44-94) walks —
entities with their group, SM quota and augmented-graph predecessors — plus
what a real GPU needs: each entity's element range of its node's buffers.
Element counts are load x ``unit_elems`` (one time unit of work for one SM);
the split segments of a node take consecutive sub-ranges in chain order, the
parallel segment rounded down so it still ends within its group's response
(SURVEY.md §7 hard part 5), so every node's full range is processed exactly
once and its output can be checked element by element.

Baselines share the same kernels and graph machinery:
  serial       one chain in topological order, each node at min(m^max, M)
  multistream  original DAG edges only, each node at min(m^max, M) — the
               naive multi-stream Greedy of PAPER.md:533 (simulate_greedy,
               simulator.cpp:96-190, run by the hardware scheduler)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _abi
from ._lib import check, lib

WL_MIX32, WL_AXPY32, WL_MIX32_TMA, WL_MIX32_LDG8 = 0, 1, 3, 4
BYTES_PER_ELEM = {WL_MIX32: 8, WL_AXPY32: 12, WL_MIX32_TMA: 8, WL_MIX32_LDG8: 8}
# ds_exec_plan.barrier_groups (include/dagsched_b200.h DS_PLAN_*)
PLAN_DEPS, PLAN_BARRIERS, PLAN_PRIORITY = 0, 1, 2


class ds_exec_entity(C.Structure):
    _fields_ = [("group", C.c_int32), ("parallelism", C.c_int32), ("node", C.c_int32),
                ("pred_off", C.c_uint32), ("n_preds", C.c_uint32), ("reserved", C.c_uint32),
                ("elem_lo", C.c_uint64), ("elem_hi", C.c_uint64)]


class ds_exec_plan(C.Structure):
    _fields_ = [("n_entities", C.c_int32), ("n_nodes", C.c_int32), ("entities", C.c_void_p),
                ("preds", C.c_void_p), ("node_elems", C.c_void_p), ("barrier_groups", C.c_int32),
                ("reserved", C.c_int32)]


class ds_exec_cfg(C.Structure):
    _fields_ = [("workload", C.c_int32), ("block_threads", C.c_int32), ("seed", C.c_uint32),
                ("sm_limit", C.c_int32), ("engine", C.c_int32), ("chunk_elems", C.c_int32)]


ENGINE_GRAPH, ENGINE_GRAPH_FREE, ENGINE_DYNAMIC, ENGINE_STREAMS = 0, 2, 3, 5
FREE_CTA_FACTOR = 4  # DS_FREE_CTA_FACTOR


class ds_exec_trace(C.Structure):
    _fields_ = [("span", C.c_void_p), ("stamps", C.c_void_p), ("smids", C.c_void_p), ("launch_ms", C.c_void_p)]


def _sig():
    L = lib()
    if getattr(L, "_exec_sig", False):
        return L
    P = C.POINTER
    for name, res, args in (
        ("ds_exec_create", C.c_int, [P(ds_exec_plan), P(ds_exec_cfg), C.c_int, P(C.c_void_p)]),
        ("ds_exec_run", C.c_int, [C.c_void_p, C.c_int, C.c_int, P(ds_exec_trace)]),
        ("ds_exec_total_ctas", C.c_int, [C.c_void_p, P(C.c_uint64)]),
        ("ds_exec_sm_count", C.c_int, [C.c_void_p, P(C.c_int)]),
        ("ds_exec_read_output", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]),
        ("ds_exec_free", C.c_int, [C.c_void_p]),
        ("ds_node_kernel_bench", C.c_int, [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, P(C.c_float),
                                           P(C.c_uint64), C.c_int]),
    ):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    L._exec_sig = True
    return L


# ------------------------------------------------------------------ plans
@dataclass
class PlanEntity:
    name: str
    group: int
    parallelism: int
    node: int
    preds: list
    lo: int
    hi: int
    exec_units: Fraction  # modelled duration (time units)


@dataclass
class Plan:
    entities: list
    node_elems: list
    barrier_groups: int  # PLAN_DEPS / PLAN_BARRIERS / PLAN_PRIORITY (a bool reads as DEPS / BARRIERS)
    bound_units: Fraction | None = None  # Theorem-1 bound, time units
    n_groups: int = 0

    def to_c(self):
        ents = (ds_exec_entity * len(self.entities))()
        preds = []
        for i, e in enumerate(self.entities):
            ents[i] = ds_exec_entity(e.group, e.parallelism, e.node, len(preds), len(e.preds), 0, e.lo, e.hi)
            preds.extend(e.preds)
        pa = (C.c_uint32 * max(1, len(preds)))(*preds)
        ne = (C.c_uint64 * len(self.node_elems))(*self.node_elems)
        plan = ds_exec_plan(len(self.entities), len(self.node_elems), C.addressof(ents), C.addressof(pa),
                            C.addressof(ne), int(self.barrier_groups), 0)  # bool -> DEPS / BARRIERS
        plan._keep = (ents, pa, ne)
        return plan


def node_elements(loads, unit_elems: int):
    return [max(4, int(Fraction(l) * unit_elems)) for l in loads]


def plan_from_scheme(scheme, loads, unit_elems: int, barrier_groups: bool = True, mode: int | None = None) -> Plan:
    """The proposed schedule (scheme.Scheme from ds_schedule_batch).

    mode PLAN_BARRIERS (barrier_groups=True): the augmented graph plus group
    barriers (simulate_scheme semantics); PLAN_DEPS (barrier_groups=False):
    the augmented graph alone (original edges + extra dependencies Ē);
    PLAN_PRIORITY: the precedence edges alone (original edges resolved to
    segment chains, Ē dropped) — the dynamic engine then enforces the group
    order by claim priority (include/dagsched_b200.h DS_PLAN_PRIORITY)."""
    if mode is None:
        mode = PLAN_BARRIERS if barrier_groups else PLAN_DEPS
    extra = set(scheme.extra_deps) if mode == PLAN_PRIORITY else set()
    elems = node_elements(loads, unit_elems)
    ordered = []  # group order; launches then members (creation order)
    for g in scheme.groups:
        ordered.extend(g.launches)
        ordered.extend(g.members)
    index = {e.id: i for i, e in enumerate(ordered)}
    cursor = [0] * len(loads)
    chain_left = {}
    for e in ordered:  # entities of one origin, in chain order
        chain_left[e.id.origin] = chain_left.get(e.id.origin, 0) + 1
    ents = []
    for e in ordered:
        v = e.id.origin
        chain_left[v] -= 1
        if chain_left[v] == 0:
            lo, hi = cursor[v], elems[v]  # the chain's last entity takes the rest
        else:
            n = int(Fraction(e.load) / Fraction(loads[v]) * elems[v])  # rounded down
            lo, hi = cursor[v], cursor[v] + n
        cursor[v] = hi
        preds = [index[p] for p in e.preds if (p, e.id) not in extra]
        ents.append(PlanEntity(str(e.id), e.group, e.parallelism, v, preds, lo, hi, e.exec))
    return Plan(ents, elems, int(mode), scheme.bounds["proposed"], len(scheme.groups))


def topo_order(n, edges):
    indeg = [0] * n
    succ = [[] for _ in range(n)]
    for u, v in edges:
        succ[u].append(v)
        indeg[v] += 1
    q = [i for i in range(n) if indeg[i] == 0]
    out = []
    while q:
        u = q.pop(0)
        out.append(u)
        for v in sorted(succ[u]):
            indeg[v] -= 1
            if indeg[v] == 0:
                q.append(v)
    return out


def _mmax(load, tmin=Fraction(1)):
    return max(1, int(Fraction(load) / tmin))


def plan_baseline(kind: str, loads, edges, sm_count: int, unit_elems: int) -> Plan:
    """'serial' (one stream) or 'multistream' (original edges) at m = min(m^max, M)."""
    n = len(loads)
    elems = node_elements(loads, unit_elems)
    order = topo_order(n, edges)
    pos = {v: i for i, v in enumerate(order)}
    preds = [[] for _ in range(n)]
    for u, v in edges:
        preds[v].append(u)
    ents = []
    for i, v in enumerate(order):
        m = min(_mmax(loads[v]), sm_count)
        if kind == "serial":
            pr = [i - 1] if i else []
        elif kind == "multistream":
            pr = sorted(pos[u] for u in preds[v])
        else:
            raise ValueError(kind)
        ex = max(Fraction(1), Fraction(loads[v]) * ((m + sm_count - 1) // sm_count) / m)
        ents.append(PlanEntity(str(v), -1, m, v, pr, 0, elems[v], ex))
    return Plan(ents, elems, PLAN_DEPS)


# ------------------------------------------------------------------ running
@dataclass
class RunResult:
    makespan_us: np.ndarray   # [replays] device-timed (globaltimer), first CTA start -> last CTA end
    launch_ms: np.ndarray     # [replays] CUDA-event time around each graph launch
    stamps: np.ndarray | None  # [replays, total_ctas, 2] ns
    smids: np.ndarray | None   # [replays, total_ctas]


class Executor:
    def __init__(self, plan: Plan, workload: int = WL_MIX32, threads: int = 1024, seed: int = 1, device: int = 0,
                 sm_limit: int = 0, engine: int = ENGINE_GRAPH, chunk_elems: int = 0):
        """sm_limit > 0 runs inside a green context of that many SMs; engine
        ENGINE_DYNAMIC runs the plan as one resident CTA per SM claiming
        entity ranks (exact group-priority claiming for PLAN_PRIORITY plans;
        ENGINE_GRAPH runs them with per-node launch priorities instead)."""
        L = _sig()
        self.plan = plan
        self.workload = workload
        self.seed = seed
        self.h = C.c_void_p()
        self._cplan = plan.to_c()
        cfg = ds_exec_cfg(workload, threads, seed, int(sm_limit), int(engine), int(chunk_elems))
        check(L.ds_exec_create(C.byref(self._cplan), C.byref(cfg), device, C.byref(self.h)))
        t = C.c_uint64()
        check(L.ds_exec_total_ctas(self.h, C.byref(t)))
        self.total_ctas = t.value
        sms = C.c_int()
        check(L.ds_exec_sm_count(self.h, C.byref(sms)))
        self.sm_count = sms.value
        # stamp slots per entity (GRAPH_FREE launches FREE_CTA_FACTOR x parallelism CTAs)
        factor = FREE_CTA_FACTOR if engine == ENGINE_GRAPH_FREE else 1
        self.slots = np.cumsum([0] + [factor * e.parallelism for e in plan.entities])
        plan._slots = self.slots

    def run(self, replays: int, warmup: int = 3, stamps: bool = True) -> RunResult:
        span = np.zeros((replays, 2), np.uint64)
        launch = np.zeros(replays, np.float32)
        st = np.zeros((replays, self.total_ctas, 2), np.uint64) if stamps else None
        sm = np.zeros((replays, self.total_ctas), np.uint32) if stamps else None
        tr = ds_exec_trace(span.ctypes.data, st.ctypes.data if stamps else None,
                           sm.ctypes.data if stamps else None, launch.ctypes.data)
        check(_sig().ds_exec_run(self.h, warmup, replays, C.byref(tr)))
        mk = (span[:, 1] - span[:, 0]).astype(np.float64) / 1e3
        return RunResult(mk, launch, st, sm)

    def output(self, node: int) -> np.ndarray:
        n = self.plan.node_elems[node]
        out = np.zeros(n, np.uint32)
        check(_sig().ds_exec_read_output(self.h, node, out.ctypes.data, n))
        return out

    def close(self):
        if self.h:
            _sig().ds_exec_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ host twins
def mix32(v: np.ndarray) -> np.ndarray:
    """Host twin of k2_workload.cuh mix32 (lowbias32)."""
    v = v.astype(np.uint32)
    v ^= v >> np.uint32(16)
    v = (v * np.uint32(0x7FEB352D)).astype(np.uint32)
    v ^= v >> np.uint32(15)
    v = (v * np.uint32(0x846CA68B)).astype(np.uint32)
    v ^= v >> np.uint32(16)
    return v


def node_input(seed: int, node: int, n: int) -> np.ndarray:
    """Host twin of k2_init for the uint32 workloads."""
    s = np.uint32((seed * 0x9E3779B9 + node) & 0xFFFFFFFF)
    i = np.arange(n, dtype=np.uint64)
    hi = (i >> np.uint64(32)).astype(np.uint32)
    key = mix32(s ^ (hi * np.uint32(0x9E3779B9)).astype(np.uint32))
    return mix32(i.astype(np.uint32) ^ key)


def node_inputs_fp(seed: int, node: int, n: int):
    h = node_input(seed, node, n)
    x = ((h >> np.uint32(8)).astype(np.int64) - (1 << 23)).astype(np.float32) * np.float32(1.0 / (1 << 23))
    y = ((mix32(h) >> np.uint32(8)).astype(np.int64) - (1 << 23)).astype(np.float32) * np.float32(1.0 / (1 << 23))
    return x, y


# ------------------------------------------------------------------ checks
def entity_windows(plan: Plan, res: RunResult, r: int):
    st = res.stamps[r]
    win = []
    for i in range(len(plan.entities)):
        s = st[plan_slots(plan)[i]:plan_slots(plan)[i + 1]]
        win.append((int(s[:, 0].min()), int(s[:, 1].max())))
    return win


def plan_slots(plan: Plan):
    if not hasattr(plan, "_slots"):
        plan._slots = np.cumsum([0] + [e.parallelism for e in plan.entities])
    return plan._slots


def check_precedence(plan: Plan, res: RunResult, r: int):
    """check_precedence (simulator.cpp:209-224) on measured stamps: no entity
    starts before every augmented predecessor has finished."""
    win = entity_windows(plan, res, r)
    bad = []
    for i, e in enumerate(plan.entities):
        for p in e.preds:
            if win[p][1] > win[i][0]:
                bad.append((plan.entities[p].name, e.name, win[p][1] - win[i][0]))
    return bad


def check_sm_exclusive(plan: Plan, res: RunResult, r: int):
    """check_capacity (simulator.cpp:192-207) at SM granularity: no two CTAs
    share an SM at the same time, i.e. every entity really held m SMs."""
    st, sm = res.stamps[r], res.smids[r]
    bad = 0
    order = np.lexsort((st[:, 0], sm))
    for a, b in zip(order[:-1], order[1:]):
        if sm[a] == sm[b] and st[b, 0] < st[a, 1]:
            bad += 1
    return bad


def group_overlap_violations(plan: Plan, res: RunResult, r: int):
    """Entities of group g+1 that started before some entity of group g ended
    (a contract of barrier plans only)."""
    if int(plan.barrier_groups) != PLAN_BARRIERS:
        return 0
    win = entity_windows(plan, res, r)
    by = {}
    for i, e in enumerate(plan.entities):
        by.setdefault(e.group, []).append(i)
    bad = 0
    for g in sorted(by):
        if g + 1 in by:
            end = max(win[i][1] for i in by[g])
            bad += sum(1 for i in by[g + 1] if win[i][0] < end)
    return bad


STALL_US = 1000.0  # a replay / sample this far above the median is a platform stall


def calibrate(unit_elems: int, sm_limit: int = 0, workload: int = WL_MIX32, replays: int = 200, groups: int = 16,
              device: int = 0):
    """Time unit and per-group latency, measured through the executor itself.

    tau: worst makespan of one entity holding every SM of the partition, each
    CTA processing one unit (full HBM contention — the most any group member
    can see). delta: worst extra latency per group boundary, from a chain of
    `groups` such groups joined by barriers. Worst = max over the samples
    without a platform stall. A schedule's bound in microseconds is then
    bound * tau + (|groups| - 1) * delta <= bound * (tau + delta), since every
    group's response is at least t_min = 1 unit.
    """
    probe = Executor(Plan([PlanEntity("u", 0, 1, 0, [], 0, 4, Fraction(1))], [4], True),
                     workload=workload, sm_limit=sm_limit, device=device)
    sms = probe.sm_count
    probe.close()
    # a barrier chain of groups over distinct buffers so that, as in a real
    # DAG, the working set (groups x sms x unit x 8 B) is DRAM- not L2-resident
    n = sms * unit_elems
    groups = max(groups, -(-(256 << 20) // (n * BYTES_PER_ELEM[workload])))
    reps = max(20, replays // 4)
    chain = Plan([PlanEntity(f"g{g}", g, sms, g, [], 0, n, Fraction(1)) for g in range(groups)], [n] * groups, True)
    ex = Executor(chain, workload=workload, sm_limit=sm_limit, device=device)
    rc = ex.run(reps, warmup=3, stamps=True)
    ex.close()
    dur, gap = [], []
    for r in range(reps):
        w = entity_windows(chain, rc, r)
        dur += [(b - a) / 1e3 for a, b in w]
        gap += [(w[g + 1][0] - w[g][1]) / 1e3 for g in range(groups - 1)]
    # worst case over the calibration samples (a real-time bound wants the
    # WCET, not a percentile), leaving out platform stalls: samples >= 1 ms
    # above the median, which hit every engine alike (tools/stall_probe.py)
    def wc(xs):
        xs = np.asarray(xs, np.float64)
        return float(xs[xs <= np.median(xs) + STALL_US].max())

    tau, delta = wc(dur), wc(gap)
    # launch stagger: the same chain with k = 8 entities of sms/8 SMs per group
    k = min(8, sms)
    eps = 0.0
    if k > 1:
        per = sms // k
        wide = Plan([PlanEntity(f"g{g}e{j}", g, per, g * k + j, [], 0, per * unit_elems, Fraction(1))
                     for g in range(groups) for j in range(k)], [per * unit_elems] * (groups * k), True)
        ex = Executor(wide, workload=workload, sm_limit=sm_limit, device=device)
        rw = ex.run(reps, warmup=3, stamps=True)
        ex.close()
        stag = []
        for r in range(reps):
            w = entity_windows(wide, rw, r)
            for g in range(groups):
                starts = [w[g * k + j][0] for j in range(k)]
                stag.append((max(starts) - min(starts)) / 1e3 / (k - 1))
                if g + 1 < groups:  # barrier latency after a k-wide group
                    end = max(w[g * k + j][1] for j in range(k))
                    gap.append((min(w[(g + 1) * k + j][0] for j in range(k)) - end) / 1e3)
        eps = wc(stag)
        delta = wc(gap)
    return {"sm_count": sms, "tau_us": tau, "tau_p50_us": float(np.median(dur)), "delta_us": delta,
            "delta_p50_us": float(np.median(gap)), "eps_us": eps, "groups": groups,
            "working_set_mb": groups * n * BYTES_PER_ELEM[workload] / 2 ** 20}


def bound_us(scheme, cal) -> float:
    """Theorem-1 bound in microseconds on this box: every group costs its
    response in time units plus the measured group-boundary latency delta and
    a launch stagger eps per additional concurrent entity."""
    total = 0.0
    for j, g in enumerate(scheme.groups):
        k = len(g.members) + len(g.launches)
        total += float(g.response) * cal["tau_us"] + (k - 1) * cal.get("eps_us", 0.0)
        if j:
            total += cal["delta_us"]
    return total


def node_kernel_bench(workload: int, ctas: int, elems_per_cta: int, reps: int = 20, threads: int = 1024,
                      device: int = 0):
    """-> (ms per launch [CUDA events], globaltimer span ns of one launch)."""
    ms = C.c_float()
    span = C.c_uint64()
    check(_sig().ds_node_kernel_bench(workload, ctas, elems_per_cta, threads, reps, C.byref(ms), C.byref(span),
                                      device))
    return ms.value, span.value

"""Schedules from the device: ds_schedule_batch + host materialisation.

The K1 kernel (csrc/k1_analysis.cuh, DETAIL mode) computes the whole of
``schedule()`` (scheduler.cpp:175-427) on the GPU and emits, per DAG, the
entity records in creation order, the executed-group records and the
division / block index of every node. What remains on the host is the
reference's *materialise* step (scheduler.cpp:361-385): replaying which
entity-level dependencies were attached to each pending entry, resolving
origin predecessors to the last segment of the origin's chain, and
collecting the extra dependency edges. ``to_reference_json`` emits exactly
the structure of the reference's ``write_scheme`` (task_io.cpp:94-148) so a
schedule can be compared field by field with the reference's own output.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _abi
from ._lib import check, lib, platform
from .batch import DagBatch, combine_status


@dataclass(frozen=True, order=True)
class EntityId:  # scheduler.hpp:19-27 (ordered by origin, generation, part)
    origin: int
    generation: int = 0
    part: int = 0  # 0 whole, 1 parallel, 2 residual

    def __str__(self):  # scheduler.cpp:9-17
        if self.part == 1:
            return f"{self.origin}:p{self.generation}"
        if self.part == 2:
            return f"{self.origin}:r{self.generation}"
        return str(self.origin)


@dataclass
class Entity:
    id: EntityId
    load: Fraction
    parallelism: int
    exec: Fraction
    group: int
    launched: bool
    preds: list = field(default_factory=list)
    residual_load: Fraction | None = None


@dataclass
class Group:
    index: int
    members: list  # [Entity]
    launches: list  # [Entity]
    spare_sms: int
    response: Fraction
    bottleneck: EntityId
    div_group: int


@dataclass
class Scheme:
    sm_count: int
    t_min: Fraction
    groups: list
    segmentations: list
    extra_deps: list
    entities: list  # sorted by id
    node_block: list
    node_div_group: list
    n_div_groups: int
    bounds: dict
    node_ids: list | None = None  # original node id of each local index (None: ids = indices)

    def entity(self, eid: EntityId) -> Entity:
        for e in self.entities:
            if e.id == eid:
                return e
        raise KeyError(str(eid))


def _q(n, d) -> Fraction:
    return Fraction(int(n), int(d))


def _fs(q: Fraction) -> str:  # format_exact (rational.cpp:87-91)
    return str(q.numerator) if q.denominator == 1 else f"{q.numerator}/{q.denominator}"


def schedule_batch(batch: DagBatch, sm_count: int, t_min=1, device: int = 0, min_load=None):
    """Run ds_schedule_batch -> list of Scheme (None where status != OK), status.

    Entities are kept in local-index space (origin = rank of the node id, what
    the executor indexes by); ``Scheme.node_ids`` maps them back to the task's
    ids for ``to_reference_json``. min_load: see ``_lib.platform``."""
    n, N = batch.n_dags, batch.n_nodes
    st = np.zeros(n, np.int32)
    ne = np.zeros(n, np.uint16)
    ng = np.zeros(n, np.uint16)
    nd = np.zeros(n, np.uint16)
    nb = np.zeros(max(N, 1), np.int16)
    ndg = np.zeros(max(N, 1), np.int16)
    ents = (_abi.ds_entity_rec * max(2 * N, 1))()
    grps = (_abi.ds_group_rec * max(N, 1))()
    bnd = np.zeros((n, 10), np.int64)
    # unlaunched-candidate masks: n_d * ceil(n_d / 64) words per DAG (header layout)
    sizes = np.diff(batch.node_off.astype(np.int64))
    ubase = np.concatenate([[0], np.cumsum(sizes * ((sizes + 63) // 64))]).astype(np.int64)
    unl = np.zeros(max(int(ubase[-1]), 1), np.uint64)
    out = _abi.ds_scheme_out(st.ctypes.data, ne.ctypes.data, ng.ctypes.data, nd.ctypes.data,
                             nb.ctypes.data, ndg.ctypes.data, C.addressof(ents), C.addressof(grps),
                             bnd.ctypes.data, unl.ctypes.data)
    cb = batch.as_c()
    pl = platform(sm_count, t_min, min_load)
    check(lib().ds_schedule_batch(C.byref(cb), C.byref(pl), C.byref(out), device))
    status = combine_status(batch.pack_status, st)
    tmin = Fraction(t_min)
    schemes = []
    for d in range(n):
        if status[d] != _abi.DS_OK:
            schemes.append(None)
            continue
        # device outputs are indexed relative to node_off[0] (header contract)
        n0, n1 = int(batch.node_off[d] - batch.node_off[0]), int(batch.node_off[d + 1] - batch.node_off[0])
        e0, e1 = int(batch.edge_off[d] - batch.edge_off[0]), int(batch.edge_off[d + 1] - batch.edge_off[0])
        succ = [[] for _ in range(n1 - n0)]
        pred = [[] for _ in range(n1 - n0)]
        for w in batch.edges[e0:e1]:
            u, v = int(w) >> 16, int(w) & 0xFFFF
            succ[u].append(v)
            pred[v].append(u)
        schemes.append(_materialise(
            sm_count, tmin, [ents[2 * n0 + i] for i in range(int(ne[d]))],
            [grps[n0 + i] for i in range(int(ng[d]))], pred, succ,
            [int(x) for x in nb[n0:n1]], [int(x) for x in ndg[n0:n1]], int(nd[d]), bnd[d],
            unl[ubase[d]:ubase[d + 1]]))
        if batch.node_ids is not None:
            schemes[-1].node_ids = list(batch.node_ids[d])
    return schemes, status


def _materialise(M, tmin, erecs, grecs, pred, succ, node_block, node_div, n_div, brow, unl) -> Scheme:
    """Replay of scheduler.cpp:286-385 bookkeeping over the device records
    (``unl``: this DAG's unlaunched-candidate masks, ceil(n/64) words per group)."""
    n = len(pred)
    uw = (n + 63) // 64
    ents = []
    for r in erecs:
        e = Entity(EntityId(r.origin, r.generation, r.part), _q(r.load_num, r.load_den), r.parallelism,
                   _q(r.exec_num, r.exec_den), r.group, bool(r.launched))
        if r.part == 1:
            e.residual_load = _q(r.res_num, r.res_den)
        ents.append(e)
    eps = [[] for _ in range(n)]  # pending entity preds: (EntityId, extra)
    rec_eps = {}
    chain = [[] for _ in range(n)]
    groups, segs = [], []
    for gi, g in enumerate(grecs):
        first, nl, nm = g.first_entity, g.n_launches, g.n_members
        launches = ents[first:first + nl]
        members = ents[first + nl:first + nl + nm]
        bott = ents[g.bottleneck].id
        for e in launches:
            c = e.id.origin
            rec_eps[e.id] = list(eps[c])
            chain[c].append(e.id)
            if e.id.part == 1:
                res = EntityId(c, e.id.generation, 2)
                # SegmentationRecord::source aliases the residual (scheduler.cpp:318-328)
                segs.append(dict(source=res, parallel=e.id, residual=res, parallel_load=e.load,
                                 residual_load=e.residual_load, group=gi))
                eps[c].append((e.id, False))
        for e in launches:  # scheduler.cpp:336-341
            for s in succ[bott.origin]:
                eps[s].append((e.id, True))
        mask = sum(int(unl[gi * uw + k]) << (64 * k) for k in range(uw))
        for c in range(n):  # scheduler.cpp:342-346
            if (mask >> c) & 1:
                eps[c].append((bott, True))
        for e in members:
            rec_eps[e.id] = list(eps[e.id.origin])
            chain[e.id.origin].append(e.id)
        groups.append(Group(gi, members, launches, int(g.spare_sms), _q(g.resp_num, g.resp_den), bott,
                            int(g.div_group)))
    extra = set()
    for e in ents:  # scheduler.cpp:365-385
        ps = {chain[o][-1] for o in pred[e.id.origin]}
        for p, x in rec_eps[e.id]:
            ps.add(p)
            if x:
                extra.add((p, e.id))
        e.preds = sorted(ps)
    bounds = {name: (None if int(brow[2 * k + 1]) == 0 else _q(brow[2 * k], brow[2 * k + 1]))
              for k, name in enumerate(_abi.BOUND_NAMES)}
    s = Scheme(M, tmin, groups, segs, sorted(extra), sorted(ents, key=lambda e: e.id), node_block,
               node_div, n_div, bounds)
    verify(s)
    return s


def verify(s: Scheme) -> None:
    """The reference's closing self-checks (scheduler.cpp:389-424): the
    augmented graph is acyclic and no group holds more than M SMs; a failure
    is a scheduler bug (logic_error there, DS_EINVARIANT here)."""
    from ._lib import DagschedError
    idx = {e.id: i for i, e in enumerate(s.entities)}
    indeg = [0] * len(s.entities)
    succ = [[] for _ in s.entities]
    for i, e in enumerate(s.entities):
        for p in e.preds:
            if p not in idx:
                raise DagschedError(_abi.DS_EINVARIANT, f"entity predecessor {p} is not an entity")
            succ[idx[p]].append(i)
            indeg[i] += 1
    queue = [i for i, d in enumerate(indeg) if d == 0]
    for u in queue:
        for v in succ[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                queue.append(v)
    if len(queue) != len(s.entities):
        raise DagschedError(_abi.DS_EINVARIANT, "augmented dependency graph has a cycle")
    for g in s.groups:
        if sum(m.parallelism for m in g.members) + sum(l.parallelism for l in g.launches) > s.sm_count:
            raise DagschedError(_abi.DS_EINVARIANT, "group allocation exceeds the device")


def to_reference_json(s: Scheme) -> dict:
    """The reference's write_scheme() structure (task_io.cpp:94-148), entities
    named by node id (to_string, scheduler.cpp:9-17)."""
    def ent(e):
        o = s.node_ids[e.origin] if s.node_ids is not None else e.origin
        return str(EntityId(o, e.generation, e.part))
    return {
        "platform": {"sm_count": s.sm_count, "t_min": _fs(s.t_min)},
        "groups": [{
            "index": g.index,
            "members": [{"entity": ent(m.id), "load": _fs(m.load), "parallelism": m.parallelism,
                         "exec_time": _fs(m.exec)} for m in g.members],
            "spare_sms": g.spare_sms,
            "spare_capacity": _fs(g.response * g.spare_sms),
            "response": _fs(g.response),
            "bottleneck": ent(g.bottleneck),
            "launches": [{"entity": ent(l.id), "parallelism": l.parallelism, "duration": _fs(l.exec)}
                         for l in g.launches],
        } for g in s.groups],
        "segmentations": [{"source": ent(x["source"]), "parallel": ent(x["parallel"]),
                           "residual": ent(x["residual"]), "parallel_load": _fs(x["parallel_load"]),
                           "residual_load": _fs(x["residual_load"]), "group": x["group"]}
                          for x in s.segmentations],
        "extra_deps": [[ent(a), ent(b)] for a, b in s.extra_deps],
        "entities": [{"id": ent(e.id), "load": _fs(e.load), "parallelism": e.parallelism,
                      "exec_time": _fs(e.exec), "group": e.group, "launched": e.launched,
                      "preds": [ent(p) for p in e.preds]} for e in s.entities],
    }

"""Simulator — simulator.hpp:1-70, simulator.cpp:1-224.

* ``simulate_greedy_batch`` — K6 (csrc/k6_greedy.cuh): simulate_greedy for
  every DAG of a batch x `runs` random-policy seeds, exact rational makespans
  (and optionally per-node start/finish) on the GPU.
* ``simulate_greedy`` — one DAG's SimTrace, through the same kernel (events).
* ``simulate_scheme`` — one schedule's SimTrace (host bookkeeping over the
  device-computed ScheduleScheme: each group starts when the previous one's
  members and launches have finished; simulator.cpp:44-94). The batched,
  measured form of this is K4 (``_lib.validate``).
* ``check_capacity`` / ``check_precedence`` (simulator.cpp:192-224).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional

import numpy as np

from . import _abi
from ._lib import DagschedError, check, lib, platform
from .batch import DagBatch, pack

K_SCALE_GRID = 1024  # simulator.cpp:11


@dataclass
class TimeModel:
    """TimeModel (simulator.hpp:18-24)."""
    scaled: bool = False
    seed: int = 0
    scale_min: Fraction = Fraction(1)
    scale_max: Fraction = Fraction(1)

    def bounds(self):
        """FactorSource (simulator.cpp:16-34): the 1/1024 grid bounds."""
        if not self.scaled:
            return 1024, 1024
        smin, smax = Fraction(self.scale_min), Fraction(self.scale_max)
        if smin <= 0 or smax > 1 or smin > smax:
            raise DagschedError(_abi.DS_EINVAL, "scale factors must satisfy 0 < min <= max <= 1")
        lo = max(1, math.ceil(smin * K_SCALE_GRID))
        hi = max(lo, math.floor(smax * K_SCALE_GRID))
        return lo, hi


@dataclass
class SimEvent:  # simulator.hpp:34-39
    entity: str
    start: Fraction
    finish: Fraction
    sms_held: int = 0


@dataclass
class SimTrace:  # simulator.hpp:41-44
    events: list = field(default_factory=list)
    makespan: Fraction = Fraction(0)


# ----------------------------------------------------------- std::mt19937_64
class _Mt64:
    """libstdc++ mt19937_64 + uniform_int_distribution<long long> (the host
    copy of csrc/rng.cuh, for single-trace bookkeeping)."""
    N, M = 312, 156

    def __init__(self, seed: int):
        m = [0] * self.N
        m[0] = seed & 0xFFFFFFFFFFFFFFFF
        for k in range(1, self.N):
            m[k] = (6364136223846793005 * (m[k - 1] ^ (m[k - 1] >> 62)) + k) & 0xFFFFFFFFFFFFFFFF
        self.mt, self.i = m, self.N

    def next(self) -> int:
        if self.i >= self.N:
            up, lo, a = 0xFFFFFFFFFFFFFFFF ^ ((1 << 31) - 1), (1 << 31) - 1, 0xB5026F5AA96619E9
            mt = self.mt
            for k in range(self.N):
                x = (mt[k] & up) | (mt[(k + 1) % self.N] & lo)
                mt[k] = mt[(k + self.M) % self.N] ^ (x >> 1) ^ (a if x & 1 else 0)
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF

    def uniform(self, lo: int, hi: int) -> int:
        rng = hi - lo + 1
        prod = self.next() * rng
        low = prod & 0xFFFFFFFFFFFFFFFF
        if low < rng:
            thr = (-rng) % rng
            while low < thr:
                prod = self.next() * rng
                low = prod & 0xFFFFFFFFFFFFFFFF
        return (prod >> 64) + lo


class _Factors:
    def __init__(self, tm: TimeModel):
        self.tm = tm
        self.lo, self.hi = tm.bounds()
        self.rng = _Mt64(tm.seed)

    def next(self) -> Fraction:
        if not self.tm.scaled:
            return Fraction(1)
        return Fraction(self.rng.uniform(self.lo, self.hi), K_SCALE_GRID)


# ------------------------------------------------------------------ scheme
def _label(eid, ids):
    o = ids[eid.origin] if ids is not None else eid.origin
    return f"{o}:p{eid.generation}" if eid.part == 1 else f"{o}:r{eid.generation}" if eid.part == 2 else str(o)


def simulate_scheme(scheme, time_model: Optional[TimeModel] = None, ids=None) -> SimTrace:
    """simulate_scheme (simulator.cpp:44-94) over a device-computed scheme;
    `ids` maps local indices to node ids (default: identity). Runs the
    reference's dependency audit and check_capacity."""
    tm = time_model or TimeModel()
    factors = _Factors(tm)
    tr = SimTrace()
    finish = {}
    clock = Fraction(0)
    for g in scheme.groups:
        end = clock
        for m in g.members:
            dur = m.exec * factors.next()
            tr.events.append(SimEvent(_label(m.id, ids), clock, clock + dur, m.parallelism))
            finish[m.id] = clock + dur
            end = max(end, clock + dur)
        for l in g.launches:
            dur = l.exec * factors.next()
            tr.events.append(SimEvent(_label(l.id, ids), clock, clock + dur, l.parallelism))
            finish[l.id] = clock + dur
            end = max(end, clock + dur)
        clock = end
    tr.makespan = clock
    start = {e.entity: e.start for e in tr.events}
    for ent in scheme.entities:
        s = start[_label(ent.id, ids)]
        for p in ent.preds:
            if finish[p] > s:
                raise DagschedError(_abi.DS_EINVARIANT, f"entity {_label(ent.id, ids)} started before predecessor "
                                                        f"{_label(p, ids)} finished")
    check_capacity(tr, scheme.sm_count)
    return tr


def check_capacity(trace: SimTrace, sm_count: int) -> None:
    """simulator.cpp:192-207: usage at every event start <= M."""
    for e in trace.events:
        used = sum(o.sms_held for o in trace.events if o.start <= e.start < o.finish)
        if used > sm_count:
            raise DagschedError(_abi.DS_EINVARIANT, f"SM capacity exceeded at t={e.start}")


def check_precedence(trace: SimTrace, scheme, ids=None) -> None:
    """simulator.cpp:209-224."""
    by = {e.entity: e for e in trace.events}
    for ent in scheme.entities:
        name = _label(ent.id, ids)
        if name not in by:
            raise DagschedError(_abi.DS_EINVARIANT, f"entity missing from trace: {name}")
        for p in ent.preds:
            if by[_label(p, ids)].finish > by[name].start:
                raise DagschedError(_abi.DS_EINVARIANT, f"precedence violated: {_label(p, ids)} -> {name}")


# ------------------------------------------------------------- greedy (K6)
def simulate_greedy_batch(batch: DagBatch, sm_count: int, runs: int = 1, policy: str = "random",
                          policy_seed: int = 0, time_model: Optional[TimeModel] = None, t_min=1,
                          events: bool = False, device: int = 0):
    """K6: simulate_greedy for every DAG x run (policy seed policy_seed + r).

    Returns (status int32[n, runs], makespan_num int64[n, runs],
    makespan_den int64[n, runs], events int64[N, runs, 4] or None)."""
    tm = time_model or TimeModel()
    tm.bounds()  # validates the scale range like FactorSource
    smin, smax = Fraction(tm.scale_min), Fraction(tm.scale_max)
    cfg = _abi.ds_greedy_cfg(1 if policy == "random" else 0, int(runs), int(policy_seed), int(bool(tm.scaled)), 0,
                             int(tm.seed), smin.numerator, smin.denominator, smax.numerator, smax.denominator)
    if policy not in ("random", "fifo"):
        raise DagschedError(_abi.DS_EINVAL, "policy must be 'fifo' or 'random'")
    n = batch.n_dags
    st = np.zeros((n, runs), np.int32)
    mk = np.zeros((n, runs, 2), np.int64)
    ev = np.zeros((max(batch.n_nodes, 1), runs, 4), np.int64) if events else None
    cb = batch.as_c()
    pl = platform(sm_count, t_min)
    check(lib().ds_simulate_greedy_batch(C.byref(cb), C.byref(pl), C.byref(cfg), st.ctypes.data, mk.ctypes.data,
                                         ev.ctypes.data if ev is not None else None, device))
    st = np.where(batch.pack_status[:, None] != 0, batch.pack_status[:, None], st)
    return st, mk[:, :, 0], mk[:, :, 1], ev


def simulate_greedy(task, sm_count: int, t_min=1, policy: str = "fifo", policy_seed: int = 0,
                    time_model: Optional[TimeModel] = None, device: int = 0) -> SimTrace:
    """simulate_greedy (simulator.cpp:96-190) of one task -> SimTrace (events
    sorted by start, then entity name; check_capacity applied)."""
    b = pack([task.as_pack()])
    st, num, den, ev = simulate_greedy_batch(b, sm_count, 1, policy, policy_seed, time_model, t_min, events=True,
                                             device=device)
    if st[0, 0] != _abi.DS_OK:
        raise DagschedError(int(st[0, 0]), "simulate_greedy failed")
    tr = SimTrace(makespan=Fraction(int(num[0, 0]), int(den[0, 0])))
    ids = task.ids
    for k, i in enumerate(ids):
        s = ev[k, 0]
        if s[1] == 0:
            continue  # never started (cannot happen for a valid DAG)
        m = min(_max_parallelism(task.loads[k], Fraction(t_min)), sm_count)
        tr.events.append(SimEvent(str(i), Fraction(int(s[0]), int(s[1])), Fraction(int(s[2]), int(s[3])), m))
    tr.events.sort(key=lambda e: (e.start, e.entity))
    check_capacity(tr, sm_count)
    return tr


def _max_parallelism(load: Fraction, t_min: Fraction) -> int:
    """exec_model.cpp:16-23 (the SM count a greedy kernel asks for)."""
    return max(1, min(math.floor(Fraction(load) / t_min), 2**31 - 1))


def to_double(q: Fraction) -> float:
    """to_double (rational.cpp:85): double(num) / double(den)."""
    return float(q.numerator) / float(q.denominator)

"""Fixture DAGs for configs C1-C4 (BASELINE.json ``configs``).

Shapes follow the reference's test fixtures (proj/tests/test_fixtures.hpp:12-53)
plus the two authored DAGs the reference does not ship:
an Inception-style DNN inference DAG (C3) and a DAG whose kernels exceed the
SM budget (C4). Every builder returns ``(nodes, edges)`` in the form
``batch.pack`` accepts: ``nodes = [(id, load), ...]``, ``edges = [(u, v), ...]``.
"""
from __future__ import annotations

import random


def make_example_task():
    """Paper Fig. 2 (test_fixtures.hpp:12-21): loads 1,4,3,3,2,2,1 on ids 1..7."""
    nodes = [(1, 1), (2, 4), (3, 3), (4, 3), (5, 2), (6, 2), (7, 1)]
    edges = [(1, 2), (1, 3), (1, 4), (3, 5), (4, 5), (4, 6), (2, 7), (5, 7), (6, 7)]
    return nodes, edges


def make_chain(loads):
    """a -> b -> c ... (test_fixtures.hpp:24-33)."""
    return list(enumerate(loads)), [(i - 1, i) for i in range(1, len(loads))]


def make_diamond(s=1, a=1, b=1, t=1):
    """0 -> {1, 2} -> 3 (test_fixtures.hpp:36-40)."""
    return [(0, s), (1, a), (2, b), (3, t)], [(0, 1), (0, 2), (1, 3), (2, 3)]


def make_fan(n, mid_load, end_load=1):
    """source -> n middle nodes -> sink (test_fixtures.hpp:43-53). C1 is make_fan(8, 20, 1)."""
    nodes = [(0, end_load)] + [(i, mid_load) for i in range(1, n + 1)] + [(n + 1, end_load)]
    edges = [(0, i) for i in range(1, n + 1)] + [(i, n + 1) for i in range(1, n + 1)]
    return nodes, edges


def c1_fork_join():
    """Config C1: the 10-node fork-join DAG."""
    return make_fan(8, 20, 1)


def inception_dag(modules: int = 9, scale: int = 1):
    """Config C3: Inception-style inference DAG, 2 + 8*modules nodes.

    stem -> [module]*modules -> classifier, each module being the classic four
    branches fed by the previous concat: 1x1 | 1x1->3x3 | 1x1->5x5 |
    pool->1x1, joined by a concat node. Loads 1-8 time units (many small
    kernels), growing with depth like the real network's later stages.
    """
    nodes, edges = [(0, 4 * scale)], []
    prev, nid = 0, 1
    for k in range(modules):
        g = 1 + k // 3  # stage multiplier 1, 2, 3
        b1 = nid
        b2a, b2b = nid + 1, nid + 2
        b3a, b3b = nid + 3, nid + 4
        b4a, b4b = nid + 5, nid + 6
        cat = nid + 7
        loads = {b1: 2 * g, b2a: 1 * g, b2b: min(8, 3 * g + 1), b3a: 1, b3b: min(8, 2 * g + 2),
                 b4a: 1, b4b: 1 * g, cat: 1}
        for v in (b1, b2a, b2b, b3a, b3b, b4a, b4b, cat):
            nodes.append((v, loads[v] * scale))
        edges += [(prev, b1), (prev, b2a), (b2a, b2b), (prev, b3a), (b3a, b3b), (prev, b4a),
                  (b4a, b4b), (b1, cat), (b2b, cat), (b3b, cat), (b4b, cat)]
        prev, nid = cat, nid + 8
    nodes.append((nid, 3 * scale))
    edges.append((prev, nid))
    return nodes, edges


def oversized_dag(seed: int = 0, sm_count: int = 148):
    """Config C4: kernels whose m^max >= M (Rule 2 singletons) next to light
    concurrent branches, so opportunistic launch and node segmentation fire
    (division.cpp:98-113, scheduler.cpp:304-329).

    Shape: source -> {3 heavy (load 1.2-2.5 M), 6 light chains of 2} ->
    mid join -> {2 heavy, 4 light} -> sink, plus the Fig. 2 pattern scaled
    by M/4 hanging off the source so splits happen on a realistic M.
    """
    rnd = random.Random(seed)
    nodes, edges = [(0, 2)], []
    nid = 1
    first = []
    for _ in range(3):
        nodes.append((nid, rnd.randint(int(1.2 * sm_count), int(2.5 * sm_count))))
        edges.append((0, nid))
        first.append(nid)
        nid += 1
    for _ in range(6):
        a, b = nid, nid + 1
        nodes += [(a, rnd.randint(4, 30)), (b, rnd.randint(4, 30))]
        edges += [(0, a), (a, b)]
        first.append(b)
        nid += 2
    mid = nid
    nodes.append((mid, 3))
    edges += [(v, mid) for v in first]
    nid += 1
    # scaled Fig. 2 sub-DAG between source and mid
    s = max(1, sm_count // 4)
    f = {k: nid + k - 1 for k in range(1, 8)}
    for k, l in zip(range(1, 8), (1, 4, 3, 3, 2, 2, 1)):
        nodes.append((f[k], l * s))
    for u, v in [(1, 2), (1, 3), (1, 4), (3, 5), (4, 5), (4, 6), (2, 7), (5, 7), (6, 7)]:
        edges.append((f[u], f[v]))
    edges += [(0, f[1]), (f[7], mid)]
    nid += 7
    second = []
    for _ in range(2):
        nodes.append((nid, rnd.randint(sm_count, 2 * sm_count)))
        edges.append((mid, nid))
        second.append(nid)
        nid += 1
    for _ in range(4):
        nodes.append((nid, rnd.randint(5, 60)))
        edges.append((mid, nid))
        second.append(nid)
        nid += 1
    sink = nid
    nodes.append((sink, 2))
    edges += [(v, sink) for v in second]
    return nodes, edges

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


# ---------------------------------------------------------------------------
# The paper's Tables 1-2 benchmark DAG families (Gaussian
# elimination, Laplace, Stencil). The reference does not ship them
# (data/fixtures is absent, proj/tests/CMakeLists.txt:25), so they are authored
# here in their textbook shapes, each with one source and one sink
# (dag.cpp:97-108). Loads: uniform integers in avg * [1 - jitter, 1 + jitter]
# (the paper's C_avg = 4 for Table 1, 20 for Table 2), at least 1.

def _loads(count: int, avg: float, jitter: float, seed: int):
    rnd = random.Random(seed)
    lo, hi = max(1, round(avg * (1 - jitter))), max(1, round(avg * (1 + jitter)))
    return [rnd.randint(lo, hi) for _ in range(count)]


def gaussian_elimination_dag(m: int = 8, avg: float = 4, jitter: float = 0.5, seed: int = 0):
    """Gaussian elimination on an m x m matrix: step k has a pivot task T(k,k)
    and updates T(k,j), j > k; T(k,k) -> T(k,j), T(k,j) -> T(k+1,j). Source
    T(1,1), sink T(m-1,m); (m^2 + m - 2) / 2 tasks (35 at m = 8)."""
    ids = {}
    for k in range(1, m):
        ids[(k, k)] = len(ids)
        for j in range(k + 1, m + 1):
            ids[(k, j)] = len(ids)
    edges = []
    for k in range(1, m):
        for j in range(k + 1, m + 1):
            edges.append((ids[(k, k)], ids[(k, j)]))
            if k + 1 < m:
                edges.append((ids[(k, j)], ids[(k + 1, j)]))
    loads = _loads(len(ids), avg, jitter, seed)
    return [(i, loads[i]) for i in range(len(ids))], edges


def laplace_dag(n: int = 6, avg: float = 4, jitter: float = 0.5, seed: int = 0):
    """Laplace-equation wavefront on an n x n grid: (i,j) -> (i+1,j), (i,j+1).
    Source (0,0), sink (n-1,n-1); n^2 tasks (36 at n = 6)."""
    idx = lambda i, j: i * n + j  # noqa: E731
    edges = []
    for i in range(n):
        for j in range(n):
            if i + 1 < n:
                edges.append((idx(i, j), idx(i + 1, j)))
            if j + 1 < n:
                edges.append((idx(i, j), idx(i, j + 1)))
    loads = _loads(n * n, avg, jitter, seed)
    return [(i, loads[i]) for i in range(n * n)], edges


def stencil_dag(width: int = 6, depth: int = 5, avg: float = 4, jitter: float = 0.5, seed: int = 0):
    """1-D three-point stencil over `depth` time steps: (t,i) -> (t+1,i-1),
    (t+1,i), (t+1,i+1); plus a source feeding step 0 and a sink after the last
    step; width * depth + 2 tasks (32 at 6 x 5)."""
    src, sink = 0, width * depth + 1
    idx = lambda t, i: 1 + t * width + i  # noqa: E731
    edges = [(src, idx(0, i)) for i in range(width)]
    for t in range(depth - 1):
        for i in range(width):
            for d in (-1, 0, 1):
                if 0 <= i + d < width:
                    edges.append((idx(t, i), idx(t + 1, i + d)))
    edges += [(idx(depth - 1, i), sink) for i in range(width)]
    loads = _loads(width * depth + 2, avg, jitter, seed)
    return [(i, loads[i]) for i in range(width * depth + 2)], edges


def paper_benchmarks(avg: float):
    """The three Tables 1-2 families at C_avg = avg (4: Table 1, 20: Table 2)."""
    return {"gaussian": gaussian_elimination_dag(8, avg), "laplace": laplace_dag(6, avg),
            "stencil": stencil_dag(6, 5, avg)}

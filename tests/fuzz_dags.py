"""Random general DAGs (not layered like the generator's) for parity fuzzing.

Node ids are shuffled against the topological order so every "ties by id"
rule is exercised; sizes reach the n <= 256 kernel; loads may be fractional;
some DAGs are deliberately invalid.
"""
from __future__ import annotations

import random
from fractions import Fraction


def random_dag(rng: random.Random, n: int, density: float, frac: bool, tmin: Fraction, big_frac: float = 0.1,
               scale: int = 1):
    order = list(range(n))
    ids = rng.sample(range(10 * n + 5), n)  # sparse, shuffled ids
    edges = set()
    for k in range(1, n - 1):
        edges.add((order[rng.randrange(0, k)], order[k]))  # one parent among earlier nodes
        for j in range(k):
            if rng.random() < density:
                edges.add((order[j], order[k]))
    if n > 1:
        has_child = {u for u, _ in edges}
        for k in range(n - 1):
            if order[k] not in has_child:
                edges.add((order[k], order[n - 1]))
    loads = []
    for _ in range(n):
        if rng.random() < big_frac:
            base = rng.randint(50, 400)  # oversized kernels (Rule 2, splits)
        else:
            base = rng.randint(1, 40)
        l = Fraction(base, rng.choice([1, 1, 2, 3, 7])) if frac else Fraction(base)
        if scale > 1:  # wide values: the 64- and 128-bit tiers, and the 128-bit ceiling
            l = l * rng.randint(1, scale) / rng.choice([1, 1, 3, 7, 65537])
        loads.append(max(l, tmin))
    nodes = [(ids[i], loads[i]) for i in range(n)]
    return nodes, [(ids[u], ids[v]) for u, v in edges]


def corpus(seed: int, count: int, max_n: int = 96, tmin=Fraction(1)):
    rng = random.Random(seed)
    dags = []
    for _ in range(count):
        n = rng.choice([1, 2, 3, rng.randint(4, 16), rng.randint(10, 40), rng.randint(30, max_n)])
        dags.append(random_dag(rng, n, rng.choice([0.0, 0.05, 0.15, 0.4]), rng.random() < 0.4, Fraction(tmin)))
    return dags


def corpus_sized(seed: int, count: int, n_lo: int, n_hi: int, tmin=Fraction(1), scale: int = 1):
    """`count` random DAGs with n in [n_lo, n_hi] (e.g. the big-DAG classes)."""
    rng = random.Random(seed)
    return [random_dag(rng, rng.randint(n_lo, n_hi), rng.choice([0.0, 0.01, 0.03]), rng.random() < 0.4,
                       Fraction(tmin), scale=scale) for _ in range(count)]


def broken(seed: int, count: int):
    """Invalid variants: cycles, extra sources/sinks, self loops, unknown ids, low loads."""
    rng = random.Random(seed)
    out = []
    for i in range(count):
        nodes, edges = random_dag(rng, rng.randint(3, 30), 0.1, False, Fraction(1))
        ids = [v for v, _ in nodes]
        kind = i % 5
        if kind == 0 and len(edges) > 1:
            u, v = sorted(edges)[0]
            edges.append((v, u))  # 2-cycle
        elif kind == 1:
            nodes.append((max(ids) + 1, 3))  # isolated node: extra source and sink
        elif kind == 2:
            edges.append((ids[0], ids[0]))
        elif kind == 3:
            edges.append((ids[0], max(ids) + 7))
        else:
            j = rng.randrange(len(nodes))
            nodes[j] = (nodes[j][0], Fraction(1, 3))  # load below t_min
        out.append((nodes, edges))
    return out

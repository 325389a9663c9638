"""K6 (batched simulate_greedy), simulate_scheme traces and run_benchmarks
against the reference's own simulator / write_trace / write_bench_table
(tests/golden/sim.json, made by oracle/_ref)."""
import glob
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2602_20826_b200 import _abi, _lib, experiment, scheme, simulator, task_io, workloads
from paper_2602_20826_b200.batch import pack
from tests import helpers

pytestmark = pytest.mark.gpu

G = None


def golden():
    global G
    if G is None:
        with open(os.path.join(helpers.GOLDEN, "sim.json")) as f:
            G = json.load(f)
    return G


def _tm(c):
    return simulator.TimeModel(c["scaled"], c["time_seed"], Fraction(c["scale_min"]), Fraction(c["scale_max"]))


@pytest.mark.parametrize("k", range(6))
def test_greedy_makespans_match_reference(k):
    c = golden()["greedy"][k]
    corp = _lib.Corpus(c["n"], **c["config"])
    st, num, den, _ = simulator.simulate_greedy_batch(corp.batch(), c["sm_count"], c["runs"], c["policy"],
                                                      c["policy_seed"], _tm(c))
    want_st = np.asarray(c["status"], np.int32)
    want = np.asarray(c["makespan"], np.int64)
    assert np.array_equal(st, want_st)
    assert np.array_equal(num, want[:, :, 0]) and np.array_equal(den, want[:, :, 1])


@pytest.mark.parametrize("k", range(6))
def test_greedy_traces_match_reference(k):
    c = golden()["greedy"][k]
    corp = _lib.Corpus(3, **c["config"])
    b = corp.batch()
    for d in range(3):
        n0, n1 = int(b.node_off[d]), int(b.node_off[d + 1])
        e0, e1 = int(b.edge_off[d]), int(b.edge_off[d + 1])
        nodes = [(i, Fraction(int(b.load_num[n0 + i]), int(b.load_den[n0 + i]))) for i in range(n1 - n0)]
        edges = [(int(w) >> 16, int(w) & 0xFFFF) for w in b.edges[e0:e1]]
        t = task_io.make_task(nodes, edges)
        tr = simulator.simulate_greedy(t, c["sm_count"], 1, c["policy"], c["policy_seed"] + 1, _tm(c))
        assert task_io.write_trace(tr) == c["traces"][d], (k, d)


def _dag(name, M):
    return {"fig2": workloads.make_example_task, "c1": workloads.c1_fork_join, "c3": workloads.inception_dag,
            "c4": lambda: workloads.oversized_dag(0, M)}[name]()


@pytest.mark.parametrize("k", range(6))
def test_scheme_traces_match_reference(k):
    c = golden()["scheme_traces"][k]
    nodes, edges = _dag(c["name"], c["sm_count"])
    b = pack([(nodes, edges)])
    schemes, st = scheme.schedule_batch(b, c["sm_count"])
    assert st[0] == 0
    # the golden's DagTask was rebuilt from the packed batch: ids = local indices
    tr = simulator.simulate_scheme(schemes[0], _tm(c))
    simulator.check_precedence(tr, schemes[0])
    assert task_io.write_trace(tr) == c["trace"]


@pytest.mark.parametrize("k", range(2))
def test_run_benchmarks_matches_reference(k):
    c = golden()["benchmarks"][k]
    paths = [os.path.join(helpers.GOLDEN, "bench_fixtures", f) for f in c["fixtures"]]
    cells = experiment.run_benchmarks(paths, c["sm_counts"], c["avg_loads"], c["greedy_runs"], c["seed"])
    assert experiment.write_bench_table(cells) == c["csv"]


def test_greedy_batch_properties_at_scale():
    """Size-independent checks on 20k DAGs x 4 runs: every run completes; the
    makespan is at least the critical-path lower bound and the greedy bound
    holds (Graham: greedy makespan <= greedy bound); fifo equals random with
    identical releases impossible to break."""
    corp = _lib.Corpus(20000, seed=123)
    b = corp.batch()
    st, num, den, _ = simulator.simulate_greedy_batch(b, 148, 4, "random", 5)
    assert (st == 0).all()
    _, bounds, _ = _lib.analyze(b, 148)
    for d in range(0, 20000, 97):
        low = Fraction(int(bounds[d, 8]), int(bounds[d, 9]))
        gb = Fraction(int(bounds[d, 2]), int(bounds[d, 3]))
        for r in range(4):
            mk = Fraction(int(num[d, r]), int(den[d, r]))
            assert low <= mk <= gb, (d, r, low, mk, gb)


def test_greedy_rejects_bad_args():
    b = pack([workloads.make_example_task()])
    with pytest.raises(_lib.DagschedError):
        simulator.simulate_greedy_batch(b, 8, 2, "random", 0, simulator.TimeModel(True, 1, Fraction(3, 4),
                                                                                   Fraction(1, 2)))
    with pytest.raises(_lib.DagschedError):
        simulator.simulate_greedy_batch(b, 8, 0)


@pytest.mark.parametrize("policy,scaled", [("random", False), ("fifo", True)])
def test_greedy_big_dags_match_reference_live(policy, scaled):
    """K6 on DAGs of ~190-940 nodes (the HBM-slot class, n > 256, and the
    64 < n <= 256 class side by side) against the reference's simulate_greedy
    on the same generated corpus, computed live by oracle/_ref."""
    from oracle import bindings
    cfgs = [dict(depth_min=16, depth_max=26, max_width=32, seed=910), dict(depth_min=26, depth_max=34, max_width=48,
                                                                           seed=911)]
    for cfg in cfgs:
        runs, M = 3, 32
        tm = simulator.TimeModel(scaled, 7, Fraction(1, 2), Fraction(1))
        corp = _lib.Corpus(6, **cfg)
        st, num, den, _ = simulator.simulate_greedy_batch(corp.batch(), M, runs, policy, 5, tm)
        rc = bindings.Checker("ref").generate(6, **cfg)
        st_r, mk_r = bindings.ref_sim_greedy(rc, M, runs, policy, 5, scaled, 7, "1/2", 1)
        assert int(corp.batch().sizes().max()) > 256
        assert np.array_equal(st, st_r), (cfg, st, st_r)
        assert np.array_equal(num, mk_r[:, :, 0]) and np.array_equal(den, mk_r[:, :, 1]), cfg

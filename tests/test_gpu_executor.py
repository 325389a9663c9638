"""GPU suite for the executor (K3) and node workloads (K2).

* node-kernel outputs are bit-exact against host twins (integer mix: exact;
  fp32 axpy: computed without FMA contraction, so numpy float32 is exact);
* measured traces satisfy the reference's executor contracts on every
  replay: check_precedence (simulator.cpp:209-224) on %globaltimer stamps,
  SM exclusivity (check_capacity, :192-207, at SM granularity) on %smid, and
  group order (simulate_scheme, :44-94) with barrier_groups.
"""
import numpy as np
import pytest

from paper_2602_20826_b200 import executor as X
from paper_2602_20826_b200 import scheme, workloads, _lib
from paper_2602_20826_b200.batch import pack

pytestmark = pytest.mark.gpu
UNIT = 4096  # small unit for tests


def _scheme_and_loads(dag, M):
    b = pack([dag])
    schemes, st = scheme.schedule_batch(b, M)
    assert st[0] == 0
    nodes = sorted(dag[0], key=lambda t: t[0]) if isinstance(dag[0][0], tuple) else list(enumerate(dag[0]))
    loads = [l for _, l in nodes]
    ids = [i for i, _ in nodes]
    idx = {i: k for k, i in enumerate(ids)}
    edges = [(idx[u], idx[v]) for u, v in dag[1]]
    return schemes[0], loads, edges


@pytest.mark.parametrize("workload", [X.WL_MIX32, X.WL_MIX32_TMA, X.WL_MIX32_LDG8])
@pytest.mark.parametrize("name,dag,M", [("fig2_M8_split", workloads.make_example_task(), 8),
                                        ("c1_fan", workloads.c1_fork_join(), 148),
                                        ("c4", workloads.oversized_dag(1, 148), 148)])
def test_outputs_bit_exact(workload, name, dag, M):
    s, loads, edges = _scheme_and_loads(dag, M)
    plan = X.plan_from_scheme(s, loads, UNIT + 3)  # odd unit: ragged slices
    ex = X.Executor(plan, workload=workload, seed=5)
    ex.run(1, warmup=0, stamps=False)
    for v in range(len(loads)):
        want = X.mix32(X.node_input(5, v, plan.node_elems[v]))
        assert np.array_equal(ex.output(v), want), (name, v)
    ex.close()


def test_axpy_matches_numpy_fp32():
    s, loads, edges = _scheme_and_loads(workloads.make_example_task(), 8)
    plan = X.plan_from_scheme(s, loads, UNIT + 1)
    ex = X.Executor(plan, workload=X.WL_AXPY32, seed=9)
    ex.run(1, warmup=0, stamps=False)
    for v in range(len(loads)):
        x, y = X.node_inputs_fp(9, v, plan.node_elems[v])
        want = (np.float32(0.75) * x) + y
        got = ex.output(v).view(np.float32)
        assert np.array_equal(got, want), v  # tolerance 0 ulp: no FMA contraction
    ex.close()


def test_segments_cover_each_node_once():
    s, loads, edges = _scheme_and_loads(workloads.make_example_task(), 8)
    assert s.segmentations, "Fig. 2 at M=8 splits node 2 (Appendix A.2)"
    plan = X.plan_from_scheme(s, loads, 1000)
    for v in range(len(loads)):
        rng = sorted((e.lo, e.hi) for e in plan.entities if e.node == v)
        assert rng[0][0] == 0 and rng[-1][1] == plan.node_elems[v]
        assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))


@pytest.mark.parametrize("barrier", [True, False])
def test_trace_contracts_hold(barrier):
    corpus = _lib.Corpus(40, seed=1)
    b = corpus.batch()
    schemes, st = scheme.schedule_batch(b, 148)
    for d in range(0, 40, 8):
        n0, n1 = int(b.node_off[d]), int(b.node_off[d + 1])
        loads = [int(x) for x in b.load_num[n0:n1]]
        plan = X.plan_from_scheme(schemes[d], loads, 8192, barrier_groups=barrier)
        ex = X.Executor(plan)
        res = ex.run(20, warmup=2)
        for r in range(20):
            assert X.check_precedence(plan, res, r) == []
            assert X.check_sm_exclusive(plan, res, r) == 0
            if barrier:
                assert X.group_overlap_violations(plan, res, r) == 0
        assert (res.makespan_us > 0).all()
        ex.close()


@pytest.mark.parametrize("kind", ["serial", "multistream"])
def test_baselines_run_and_respect_edges(kind):
    dag = workloads.inception_dag()
    loads = [l for _, l in dag[0]]
    plan = X.plan_baseline(kind, loads, dag[1], 148, 4096)
    ex = X.Executor(plan)
    res = ex.run(10, warmup=2)
    for r in range(10):
        assert X.check_precedence(plan, res, r) == []
        assert X.check_sm_exclusive(plan, res, r) == 0
    for v in (0, 5, len(loads) - 1):
        assert np.array_equal(ex.output(v), X.mix32(X.node_input(1, v, plan.node_elems[v])))
    ex.close()


def test_node_kernel_bench_sane():
    for wl in (X.WL_MIX32, X.WL_MIX32_TMA, X.WL_MIX32_LDG8, X.WL_AXPY32):
        ms, span = X.node_kernel_bench(wl, 148, 1 << 20, reps=5)
        gbs = 148 * (1 << 20) * X.BYTES_PER_ELEM[wl] / (ms * 1e-3) / 1e9
        assert 500 < gbs < 9000, (wl, gbs)
        assert span > 0


def test_green_context_partition():
    """sm_limit runs the graph inside a green context: the executor reports the
    partition size and every CTA lands on one of that many SMs."""
    s, loads, edges = _scheme_and_loads(workloads.make_fan(6, 12, 2), 16)
    plan = X.plan_from_scheme(s, loads, 4096)
    ex = X.Executor(plan, sm_limit=16)
    assert ex.sm_count == 16
    res = ex.run(5, warmup=1)
    assert len(np.unique(res.smids)) <= 16
    for r in range(5):
        assert X.check_precedence(plan, res, r) == []
        assert X.check_sm_exclusive(plan, res, r) == 0
    for v in range(len(loads)):
        assert np.array_equal(ex.output(v), X.mix32(X.node_input(1, v, plan.node_elems[v])))
    ex.close()
    cal = X.calibrate(4096, sm_limit=16, replays=20, groups=4)
    assert cal["sm_count"] == 16 and cal["tau_us"] > 0


@pytest.mark.parametrize("engine,workload,chunk", [(X.ENGINE_DYNAMIC, X.WL_MIX32, 0),
                                                   (X.ENGINE_DYNAMIC, X.WL_MIX32_TMA, 0),
                                                   (X.ENGINE_DYNAMIC, X.WL_MIX32, 1000),
                                                   (X.ENGINE_DYNAMIC, X.WL_MIX32_TMA, 4099)])
@pytest.mark.parametrize("mode", [X.PLAN_BARRIERS, X.PLAN_DEPS, X.PLAN_PRIORITY])
def test_dynamic_engine(mode, engine, workload, chunk):
    """DS_ENGINE_DYNAMIC: resident CTAs claim (entity, rank) items from a
    device-side ready queue — every item runs exactly once per replay, outputs
    bit-exact, precedence / SM-exclusivity / group-order contracts hold; with
    DS_PLAN_PRIORITY the precedence edges alone order the entities (Ē is
    replaced by the engine's group-order claiming)."""
    barrier = mode == X.PLAN_BARRIERS
    cases = [(workloads.make_example_task(), 8), (workloads.oversized_dag(2, 148), 148),
             (workloads.inception_dag(), 148), (workloads.c1_fork_join(), 148)]
    for dag, M in cases:
        s, loads, edges = _scheme_and_loads(dag, M)
        plan = X.plan_from_scheme(s, loads, UNIT + 5, mode=mode)
        if mode == X.PLAN_PRIORITY:  # no extra dependency edge is left in the plan
            extra = {(str(a), str(b)) for a, b in s.extra_deps}
            assert not any((plan.entities[p].name, e.name) in extra for e in plan.entities for p in e.preds)
        ex = X.Executor(plan, workload=workload, engine=engine, sm_limit=0 if M == 148 else 8, chunk_elems=chunk)
        res = ex.run(8, warmup=2)
        for r in range(8):
            st = res.stamps[r]
            assert (st[:, 0] > 0).all() and (st[:, 1] >= st[:, 0]).all()
            assert X.check_precedence(plan, res, r) == []
            assert X.check_sm_exclusive(plan, res, r) == 0
            if barrier:
                assert X.group_overlap_violations(plan, res, r) == 0
        for v in range(len(loads)):
            assert np.array_equal(ex.output(v), X.mix32(X.node_input(1, v, plan.node_elems[v])))
        ex.close()


def test_dynamic_engine_runs_baseline_plans():
    dag = workloads.inception_dag()
    loads = [l for _, l in dag[0]]
    for kind, engine in (("serial", X.ENGINE_DYNAMIC), ("multistream", X.ENGINE_DYNAMIC)):
        plan = X.plan_baseline(kind, loads, dag[1], 148, 4096 + 7)
        ex = X.Executor(plan, engine=engine, workload=X.WL_MIX32_TMA)
        res = ex.run(5, warmup=1)
        for r in range(5):
            assert X.check_precedence(plan, res, r) == []
            assert X.check_sm_exclusive(plan, res, r) == 0
        ex.close()


@pytest.mark.parametrize("workload", [X.WL_MIX32_TMA, X.WL_MIX32])
def test_free_launch_runs_every_workload(workload):
    """GRAPH_FREE launches 4m 256-thread CTAs without the shared-memory ring:
    the staged workloads run their plain LDG body there (same outputs)."""
    dag = workloads.make_fan(4, 6, 2)
    loads = [l for _, l in dag[0]]
    plan = X.plan_baseline("multistream", loads, dag[1], 148, UNIT + 3)
    ex = X.Executor(plan, workload=workload, engine=X.ENGINE_GRAPH_FREE)
    res = ex.run(3, warmup=1, stamps=False)
    assert (res.makespan_us > 0).all()
    for v in range(len(loads)):
        assert np.array_equal(ex.output(v), X.mix32(X.node_input(1, v, plan.node_elems[v])))
    ex.close()



@pytest.mark.parametrize("workload", [X.WL_MIX32, X.WL_MIX32_TMA])
def test_host_streams_engine(workload):
    """DS_ENGINE_STREAMS (host-launched kernels on per-entity streams with
    events): outputs bit-exact and the trace contracts hold, for a baseline
    plan and for the schedule with group barriers."""
    dag = workloads.inception_dag()
    loads = [l for _, l in dag[0]]
    plan = X.plan_baseline("multistream", loads, dag[1], 148, 4096 + 3)
    s, loads2, edges2 = _scheme_and_loads(workloads.oversized_dag(1, 148), 148)
    for pl, lds in ((plan, loads), (X.plan_from_scheme(s, loads2, 4096 + 3, barrier_groups=True), loads2)):
        ex = X.Executor(pl, workload=workload, engine=X.ENGINE_STREAMS)
        res = ex.run(4, warmup=1)
        for r in range(4):
            assert X.check_precedence(pl, res, r) == []
            assert X.check_sm_exclusive(pl, res, r) == 0
            assert X.group_overlap_violations(pl, res, r) == 0
        for v in range(len(lds)):
            assert np.array_equal(ex.output(v), X.mix32(X.node_input(1, v, pl.node_elems[v])))
        ex.close()


def test_priority_plans_need_a_priority_engine():
    """Host streams cannot express the group order: a DS_PLAN_PRIORITY plan is
    refused there instead of running without Ē (the dynamic engine claims in
    group order, the graph engine carries per-node launch priorities)."""
    s, loads, edges = _scheme_and_loads(workloads.make_example_task(), 8)
    plan = X.plan_from_scheme(s, loads, 4096, mode=X.PLAN_PRIORITY)
    for engine in (X.ENGINE_STREAMS, X.ENGINE_GRAPH_FREE):
        with pytest.raises(_lib.DagschedError):
            X.Executor(plan, engine=engine)


@pytest.mark.parametrize("workload", [X.WL_MIX32, X.WL_MIX32_TMA])
def test_graph_priority_plans(workload):
    """DS_PLAN_PRIORITY on DS_ENGINE_GRAPH: the precedence edges alone (no Ē)
    as graph edges, each kernel node at its group's launch priority
    (cudaGraphInstantiateFlagUseNodePriority). Every CTA runs once per
    replay, outputs are bit-exact, precedence and SM exclusivity hold."""
    cases = [(workloads.make_example_task(), 8), (workloads.oversized_dag(2, 148), 148),
             (workloads.inception_dag(), 148), (workloads.c1_fork_join(), 148)]
    for dag, M in cases:
        s, loads, edges = _scheme_and_loads(dag, M)
        plan = X.plan_from_scheme(s, loads, UNIT + 5, mode=X.PLAN_PRIORITY)
        ex = X.Executor(plan, workload=workload, engine=X.ENGINE_GRAPH, sm_limit=0 if M == 148 else 8)
        res = ex.run(6, warmup=2)
        for r in range(6):
            st = res.stamps[r]
            assert (st[:, 0] > 0).all() and (st[:, 1] >= st[:, 0]).all()
            assert X.check_precedence(plan, res, r) == []
            assert X.check_sm_exclusive(plan, res, r) == 0
        for v in range(len(loads)):
            assert np.array_equal(ex.output(v), X.mix32(X.node_input(1, v, plan.node_elems[v])))
        ex.close()

"""GPU parity suite for K1 (batched bound analysis) through the C-ABI.

Every result is compared with the reference's own outputs (tests/golden,
produced by the reference sources compiled in oracle/_ref) or with the
restated oracle on seeded corpora. Integer/rational work: bit-exact.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import bindings
from paper_2602_20826_b200 import _abi, _lib, scheme
from paper_2602_20826_b200.batch import pack
from tests import helpers

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    return bindings.Checker("oracle")


def test_fixtures_bounds_and_status():
    for case in helpers.fixtures():
        b = helpers.fixture_batch(case)
        ml = helpers.min_load_arg(case)
        st, bounds, _ = _lib.analyze(b, case["sm_count"], case["t_min"], min_load=ml)
        assert int(st[0]) == case["status"], case["name"]
        assert [int(x) for x in bounds[0]] == case["bounds"], case["name"]
        if "status_no_proposed" in case:  # load < t_min fails only schedule() (scheduler.cpp:177-182)
            st, bounds, _ = _lib.analyze(b, case["sm_count"], case["t_min"], mask=0x1E, min_load=ml)
            assert int(st[0]) == case["status_no_proposed"], case["name"]
            assert [int(x) for x in bounds[0]] == case["bounds_no_proposed"], case["name"]


def test_fixture_schemes_match_reference_write_scheme():
    for case in helpers.fixtures():
        if case["status"] != 0:
            continue
        b = helpers.fixture_batch(case)
        schemes, st = scheme.schedule_batch(b, case["sm_count"], case["t_min"])
        got = scheme.to_reference_json(schemes[0])
        assert helpers.normalise_scheme(got) == helpers.normalise_scheme(case["scheme"]), case["name"]


@pytest.mark.parametrize("name,tag", [("corpus_default.npz", "default"), ("corpus_variants.npz", "heavy"),
                                      ("corpus_variants.npz", "fractional"), ("corpus_variants.npz", "wide")])
def test_golden_corpora(name, tag):
    b, res, _ = helpers.corpus(name, tag)
    for M, (st_ref, b_ref) in res.items():
        st, bounds, _ = _lib.analyze(b, M)
        assert np.array_equal(st, st_ref), M
        bad = np.nonzero((bounds != b_ref).any(1))[0]
        assert len(bad) == 0, (M, bad[:5], bounds[bad[:1]], b_ref[bad[:1]])


def test_golden_schemes_group_membership_and_quotas():
    b, _, _ = helpers.corpus()
    recs = list(helpers.schemes())
    for M in (8, 32, 148):
        sub = b.slice(0, 120)
        schemes, st = scheme.schedule_batch(sub, M)
        for rec in recs:
            if rec["sm_count"] != M:
                continue
            got = scheme.to_reference_json(schemes[rec["dag"]])
            assert helpers.normalise_scheme(got) == helpers.normalise_scheme(rec["scheme"]), (M, rec["dag"])


@pytest.mark.parametrize("cfg,Ms", [
    (dict(seed=2024), (1, 2, 5, 8, 32, 64, 148, 1000)),
    (dict(seed=7, avg_load=200, max_width=12), (8, 148, 300)),
    (dict(seed=99, integer_loads=False, avg_load=5), (4, 148)),
    (dict(seed=5, t_min="1/2", avg_load=9), (6, 148)),
    (dict(seed=31, exact_mean=True, integer_loads=False, avg_load=7), (16, 148)),
    (dict(seed=13, depth_min=6, depth_max=10, max_width=24, avg_load=40), (32, 148)),  # n > 64: W=4 kernel
])
def test_seeded_corpora_vs_oracle(orc, cfg, Ms):
    n = 4000
    gen = _lib.Corpus(n, **cfg)
    b = gen.batch()
    c = orc.corpus(b, min_load=cfg.get("t_min", 1))
    for M in Ms:
        tmin = cfg.get("t_min", 1)
        st_o, b_o, _ = c.evaluate(M, tmin)
        st, bounds, _ = _lib.analyze(b, M, tmin)
        assert np.array_equal(st, st_o), M
        bad = np.nonzero((bounds != b_o).any(1))[0]
        assert len(bad) == 0, (M, bad[:5])


@pytest.mark.parametrize("cfg,Ms", [
    (dict(seed=2024), (1, 8, 148)),
    (dict(seed=7, avg_load=200, max_width=12), (8, 300)),  # u64 / u128 word tiers
    (dict(seed=99, integer_loads=False, avg_load=5), (4, 148)),
    (dict(seed=5, t_min="1/2", avg_load=9), (6, 148)),
    (dict(seed=13, depth_min=6, depth_max=10, max_width=24, avg_load=40), (32, 148)),  # n > 64
])
def test_latency_path_vs_oracle(orc, cfg, Ms):
    """Host batches of <= 64 DAGs take the one-kernel latency path (k1_small:
    zero-copy mapped buffers, in-warp 32/64/128-bit tiers); its bounds,
    statuses and (detail mode) schedules equal the oracle's and the
    throughput path's."""
    gen = _lib.Corpus(640, **cfg)
    b = gen.batch()
    tmin = cfg.get("t_min", 1)
    c = orc.corpus(b, min_load=tmin)
    for M in Ms:
        st_o, b_o, _ = c.evaluate(M, tmin)
        for lo in range(0, 640, 64):
            st, bounds, _ = _lib.analyze(b.slice(lo, lo + 64), M, tmin)
            assert np.array_equal(st, st_o[lo:lo + 64]), (M, lo)
            assert np.array_equal(bounds, b_o[lo:lo + 64]), (M, lo)
        if b.integer_loads() and b.compact16_ok():
            st, bounds, _ = _lib.analyze16(b.slice(0, 50), M, tmin)
            assert np.array_equal(st, st_o[:50]) and np.array_equal(bounds, b_o[:50])
        big, st_big = scheme.schedule_batch(b.slice(0, 130), M, tmin)  # > 64: throughput (detail arena) path
        for lo in (0, 64):
            small, st_small = scheme.schedule_batch(b.slice(lo, lo + 64), M, tmin)
            assert np.array_equal(st_small, st_big[lo:lo + 64])
            for k, sch in enumerate(small):
                if sch is not None:
                    assert scheme.to_reference_json(sch) == scheme.to_reference_json(big[lo + k]), (M, lo + k)


@pytest.mark.parametrize("cfg,Ms", [
    (dict(seed=2024), (1, 8, 148)),
    (dict(seed=7, avg_load=200, max_width=10), (8, 300)),  # u64 / u128 word tiers
    (dict(seed=21, depth_min=2, depth_max=3, max_width=2), (4, 148)),  # tiny DAGs
    (dict(seed=23, depth_min=7, depth_max=8, max_width=9), (32, 148)),  # 33..64 nodes
])
def test_triangular_wire_form_matches_wide(cfg, Ms):
    """ds_analyze_batch_tri (bit-matrix wire form, expanded on the device by
    k_widen_tri) = ds_analyze_batch on the same DAGs: throughput path, the
    latency path (<= 64 DAGs) and the multi-device split."""
    b = _lib.Corpus(30000, **cfg).batch()
    assert b.tri_ok()
    for M in Ms:
        st, bounds, ng = _lib.analyze(b, M)
        st_t, b_t, ng_t = _lib.analyze_tri(b, M)
        assert np.array_equal(st, st_t) and np.array_equal(bounds, b_t) and np.array_equal(ng, ng_t), M
        st_s, b_s, _ = _lib.analyze_tri(b.slice(100, 160), M)
        assert np.array_equal(st_s, st[100:160]) and np.array_equal(b_s, bounds[100:160])
    st_m, b_m, _ = _lib.analyze_tri(b, 148, devices=[0] * 3)
    st, bounds, _ = _lib.analyze(b, 148)
    assert np.array_equal(st_m, st) and np.array_equal(b_m, bounds)


def test_triangular_wire_form_invalid_dags():
    """Validation statuses survive the bit-matrix form: several sources or
    sinks, load 0, duplicate edges (collapse, as DagTask::make dedups)."""
    dags = [
        ([1, 2, 3], [(0, 1), (0, 2)]),            # two sinks
        ([1, 2, 3], [(0, 2), (1, 2)]),            # two sources
        ([1, 0, 3], [(0, 1), (1, 2)]),            # load 0
        ([2, 3, 4], [(0, 1), (0, 1), (1, 2)]),    # duplicate edge
        ([5], []),                                # one node
        ([1] * 64, [(i, i + 1) for i in range(63)]),  # 64-node chain
    ]
    b = pack(dags)
    assert b.tri_ok()
    st, bounds, _ = _lib.analyze(b, 8)
    st_t, b_t, _ = _lib.analyze_tri(b, 8)
    assert np.array_equal(st, st_t) and np.array_equal(bounds, b_t)
    big = pack([([1] * 65, [(i, i + 1) for i in range(64)])])
    assert not big.tri_ok()


@pytest.mark.parametrize("n_small", [3, 40000])
def test_triangular_wire_form_rejects_dags_above_64_nodes(n_small):
    """A DAG above 64 nodes in a ds_dag_batch_tri is DS_EINVAL, whether the
    batch takes the latency path or the chunked pipeline (checked per chunk
    there, here in the last chunk)."""
    import ctypes as C
    from paper_2602_20826_b200.batch import DagBatch
    b = _lib.Corpus(n_small, seed=2).batch()
    big = pack([([1] * 65, [(i, i + 1) for i in range(64)])])
    tw = lambda x: x.tri_words()  # noqa: E731
    # the triangular arrays of b + big, packed by hand (tri() refuses the big DAG)
    both = DagBatch(np.concatenate([b.node_off, b.node_off[-1] + big.node_off[1:]]).astype(np.uint32),
                    np.concatenate([b.edge_off, b.edge_off[-1] + big.edge_off[1:]]).astype(np.uint32),
                    np.concatenate([b.load_num, big.load_num]), np.concatenate([b.load_den, big.load_den]),
                    np.concatenate([b.edges, big.edges]), np.zeros(b.n_dags + 1, np.int32))
    adj_off = tw(both)
    n = both.sizes()
    ecount = np.diff(both.edge_off.astype(np.int64))
    dag = np.repeat(np.arange(both.n_dags, dtype=np.int64), ecount)
    u = (both.edges >> 16).astype(np.int64)
    v = (both.edges & 0xFFFF).astype(np.int64)
    bits = np.zeros(int(adj_off[-1]) * 32, np.bool_)
    bits[adj_off[dag].astype(np.int64) * 32 + v * (v - 1) // 2 + u] = True
    adj = np.packbits(bits, bitorder="little").view(np.uint32).copy()
    load16 = both.load_num.astype(np.uint16)
    assert int(n.max()) == 65
    cb = both.as_ctri(load16, adj_off, adj)
    st, bo, ng, r = _lib._results(both.n_dags)
    rc = _lib.lib().ds_analyze_batch_tri(C.byref(cb), C.byref(_lib.platform(148)), _abi.DS_M_ALL, C.byref(r), 0)
    assert rc == _abi.DS_EINVAL
    assert "more than 64" in _lib.lib().ds_last_error().decode()
    # the library is still usable afterwards
    st2, b2, _ = _lib.analyze_tri(b, 148)
    st1, b1, _ = _lib.analyze(b, 148)
    assert np.array_equal(st1, st2) and np.array_equal(b1, b2)


def test_method_mask_subsets(orc):
    b = _lib.Corpus(500, seed=3).batch()
    _, full, _ = _lib.analyze(b, 148)
    for mask in (1, 2, 4, 8, 16, 5, 0x1E):
        st, part, _ = _lib.analyze(b, 148, mask=mask)
        for k in range(5):
            cols = part[:, 2 * k:2 * k + 2]
            if mask >> k & 1:
                assert np.array_equal(cols, full[:, 2 * k:2 * k + 2])
            else:
                assert not cols.any()


def test_invalid_and_edge_dags():
    dags = [
        ([], []),                                          # empty
        ([(0, 1), (0, 2)], []),                            # duplicate id
        ([(0, 1), (1, 1)], [(0, 1), (1, 0)]),              # cycle
        ([(0, 1)], [(0, 0)]),                              # self loop
        ([(0, 1), (1, 1), (2, 1)], [(0, 2), (1, 2)]),      # two sources
        ([(0, 1), (1, 1), (2, 1)], [(0, 1), (0, 2)]),      # two sinks
        ([(0, "1/2")], []),                                # load below t_min
        ([(0, 5)], []),                                    # single node
        (list(range(1, 1026)), [(i, i + 1) for i in range(1024)]),  # 1025 nodes: too big
        ([(5, 3), (9, 4), (40, 2)], [(5, 9), (9, 40), (5, 40), (5, 9)]),  # sparse ids + duplicate edge
    ]
    b = pack(dags)
    st, bounds, _ = _lib.analyze(b, 4)
    assert list(st[:8]) == [_abi.DS_E_EMPTY, _abi.DS_E_DUP_ID, _abi.DS_E_CYCLE, _abi.DS_E_SELFLOOP,
                            _abi.DS_E_SOURCES, _abi.DS_E_SINKS, _abi.DS_E_LOAD, _abi.DS_OK]
    assert st[8] == _abi.DS_ETOOBIG
    assert st[9] == _abi.DS_OK
    assert not bounds[:7].any()


def test_session_and_multi_and_device_pointers():
    torch = pytest.importorskip("torch")
    b = _lib.Corpus(20000, seed=8).batch()
    st, bounds, ng = _lib.analyze(b, 148)
    s = _lib.Session(b, 148)
    for _ in range(3):
        ms = s.run()
        assert ms > 0
    st2, b2, ng2 = s.results()
    assert np.array_equal(st, st2) and np.array_equal(bounds, b2) and np.array_equal(ng, ng2)
    st3, b3, _ = _lib.analyze_multi(b, 148, devices=[0, 0, 0])
    assert np.array_equal(st, st3) and np.array_equal(bounds, b3)
    st4, b4, ng4 = _lib.analyze16_multi(b, 148, devices=[0] * min(4, _lib.device_count() * 4))
    assert np.array_equal(st, st4) and np.array_equal(bounds, b4) and np.array_equal(ng, ng4)
    if _lib.device_count() > 1:  # real devices when the box has them
        st5, b5, _ = _lib.analyze16_multi(b, 148, devices=list(range(_lib.device_count())))
        assert np.array_equal(st, st5) and np.array_equal(bounds, b5)
    dev = torch.device("cuda:0")
    t = {k: torch.from_numpy(getattr(b, k).view(np.int32) if getattr(b, k).dtype == np.uint32
                             else getattr(b, k)).to(dev) for k in ("node_off", "edge_off", "load_num", "edges")}
    out_st = torch.zeros(b.n_dags, dtype=torch.int32, device=dev)
    out_b = torch.zeros(b.n_dags * 10, dtype=torch.int64, device=dev)
    cb = _abi.ds_dag_batch(b.n_dags, t["node_off"].data_ptr(), t["edge_off"].data_ptr(), t["load_num"].data_ptr(),
                           None, t["edges"].data_ptr())
    r = _abi.ds_results(out_st.data_ptr(), out_b.data_ptr(), None)
    pl = _lib.platform(148)
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().ds_analyze_batch(C.byref(cb), C.byref(pl), _abi.DS_M_ALL, C.byref(r), 0,
                                           C.c_void_p(stream), _abi.DS_F_DEVICE_PTRS))
    torch.cuda.synchronize()
    assert np.array_equal(out_st.cpu().numpy(), st)
    assert np.array_equal(out_b.cpu().numpy().reshape(-1, 10), bounds)


def test_full_size_properties_and_sampled_parity(orc):
    """BASELINE config C5 at full size (1M DAGs, M=148): size-independent
    properties on every DAG plus oracle parity on a 20k random sample."""
    n = 1_000_000
    b = _lib.Corpus(n, seed=1).batch()
    st, bounds, ng = _lib.analyze(b, 148)
    assert (st == 0).all()
    q = lambda k: bounds[:, 2 * k].astype(np.float64) / bounds[:, 2 * k + 1]
    prop, gr, gu, gp, lo = (q(k) for k in range(5))
    assert (bounds[:, 1::2] > 0).all()
    eps = 1e-9
    assert (lo <= prop + eps).all() and (lo <= gr + eps).all() and (lo <= gp + eps).all()
    assert (gr <= gu + eps).all()
    assert (ng >= 1).all()
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(n, 20000, replace=False))
    sub = pack_subset(b, idx)
    st_o, b_o, _ = orc.corpus(sub).evaluate(148)
    assert np.array_equal(st_o, st[idx]) and np.array_equal(b_o, bounds[idx])


def pack_subset(b, idx):
    from paper_2602_20826_b200.batch import from_arrays
    no, eo, ln, ld, ed = [0], [0], [], [], []
    for d in idx:
        n0, n1, e0, e1 = b.node_off[d], b.node_off[d + 1], b.edge_off[d], b.edge_off[d + 1]
        ln.append(b.load_num[n0:n1]); ld.append(b.load_den[n0:n1]); ed.append(b.edges[e0:e1])
        no.append(no[-1] + n1 - n0); eo.append(eo[-1] + e1 - e0)
    return from_arrays(no, eo, np.concatenate(ln), np.concatenate(ld), np.concatenate(ed))


def test_compact16_wire_form_matches_wide():
    """ds_analyze_batch16 (16-bit loads/edges, widened on the device) gives the
    same statuses and bounds as ds_analyze_batch on the same DAGs."""
    corpus = _lib.Corpus(30000, seed=11)
    b = corpus.batch()
    assert b.compact16_ok()
    st, bounds, ng = _lib.analyze(b, 148)
    st16, bounds16, ng16 = _lib.analyze16(b, 148)
    assert np.array_equal(st, st16) and np.array_equal(bounds, bounds16) and np.array_equal(ng, ng16)
    st, bounds, _ = _lib.analyze(b, 32)
    st16, bounds16, _ = _lib.analyze16(b, 32)
    assert np.array_equal(st, st16) and np.array_equal(bounds, bounds16)


def test_paper_benchmark_families_vs_oracle(orc):
    """Tables 1-2 DAG families on the GPU: bounds and group structure bit-exact."""
    from paper_2602_20826_b200 import scheme, workloads
    dags = [d for avg in (4, 20) for d in workloads.paper_benchmarks(avg).values()]
    b = pack(dags)
    for M in (8, 30, 32, 148):
        st, bounds, _ = _lib.analyze(b, M)
        st_o, b_o, _ = orc.corpus(b).evaluate(M)
        assert (st == 0).all() and np.array_equal(st, st_o) and np.array_equal(bounds, b_o), M
        schemes, st2 = scheme.schedule_batch(b, M)
        c = orc.corpus(b)
        for d, s in enumerate(schemes):
            got = helpers.normalise_scheme(scheme.to_reference_json(s))
            assert got == helpers.normalise_scheme(c.scheme(d, M)), (M, d)


@pytest.mark.parametrize("kind", ["nosort", "nofast"])
def test_k1_variants_agree(kind):
    """DS_K1_SORT=0 (walks in index order) and DS_K1_FAST=0 (no fused fast
    path: every DAG through k1_front / k1_mid) give the same results as the
    default (run in a subprocess: the selection is read once per process)."""
    import json
    import os
    import subprocess
    import sys
    code = ("import json,sys; sys.path.insert(0,'.'); from paper_2602_20826_b200 import _lib; "
            "b=_lib.Corpus(20000, seed=5).batch(); st,bo,ng=_lib.analyze(b,148); st2,bo2,_=_lib.analyze(b,16); "
            "print(json.dumps([int(st.sum()), int(bo.sum() % 1000000007), int(ng.sum()), int(bo2.sum() % 1000000007)]))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for k in ("default", kind):
        env = dict(os.environ)
        if k == "nosort":
            env["DS_K1_SORT"] = "0"
        elif k == "nofast":
            env["DS_K1_FAST"] = "0"
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, check=True)
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]


def test_lane_walk_wide_platform_matches_oracle(orc):
    """M > 255 (the paper's Fig. 4 sweep reaches M = 256): 16-bit quota
    fields in the one-lane-per-DAG walk; bit-exact vs the oracle."""
    corpus = _lib.Corpus(20000, seed=9, avg_load=200, max_width=16)
    b = corpus.batch()
    for M in (256, 300, 1000):
        st, bounds, _ = _lib.analyze(b, M)
        st_o, b_o, _ = orc.corpus(b).evaluate(M)
        assert np.array_equal(st, st_o) and np.array_equal(bounds, b_o), M


def test_host_pipeline_matches_slot_streams():
    """The four-stream host pipeline (default) and the per-chunk slot streams
    (DS_PIPE=0) give the same results over every wire form, with several
    chunks (8 chunks x 25k DAGs, more chunks than stream slots reuse them)."""
    import json
    import os
    import subprocess
    import sys
    code = ("import json,sys,hashlib; sys.path.insert(0,'.'); from paper_2602_20826_b200 import _lib; "
            "b=_lib.Corpus(200000, seed=6).batch(); h=[]\n"
            "for f in (_lib.analyze, _lib.analyze16, _lib.analyze_tri):\n"
            "    st,bo,ng=f(b,148); h.append(hashlib.sha1(st.tobytes()+bo.tobytes()+ng.tobytes()).hexdigest())\n"
            "print(json.dumps(h))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_kv in ({"DS_CHUNKS": "8"}, {"DS_CHUNKS": "8", "DS_PIPE": "0"}, {"DS_CHUNKS": "12"}):
        env = dict(os.environ, **env_kv)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, check=True)
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1] == outs[2]
    assert len(set(outs[0])) == 1  # the three wire forms agree too

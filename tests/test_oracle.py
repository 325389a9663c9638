"""CPU suite: the restated oracle (oracle/src) against the reference's own
golden vectors (tests/golden, produced by the reference compiled from its
sources, see tests/golden/make_golden.py) and, when oracle/_ref is built,
directly against the reference library on fresh corpora."""
import os
import subprocess

import numpy as np
import pytest

from oracle import bindings
from tests import helpers


@pytest.fixture(scope="module")
def orc():
    if not bindings.available("oracle"):
        subprocess.run(["make", "-C", os.path.join(helpers.GOLDEN, "..", "..", "oracle"), "oracle"], check=True)
    return bindings.Checker("oracle")


def test_fixture_bounds_status_schemes(orc):
    for case in helpers.fixtures():
        b = helpers.fixture_raw_batch(case)
        c = orc.corpus(b, min_load=case.get("min_load", case["t_min"]))
        st, bounds, _ = c.evaluate(case["sm_count"], case["t_min"], parallel=False)
        assert int(st[0]) == case["status"], case["name"]
        assert [int(x) for x in bounds[0]] == case["bounds"], case["name"]
        if "status_no_proposed" in case:
            st, bounds, _ = c.evaluate(case["sm_count"], case["t_min"], mask=0x1E, parallel=False)
            assert int(st[0]) == case["status_no_proposed"], case["name"]
            assert [int(x) for x in bounds[0]] == case["bounds_no_proposed"], case["name"]
        if case["status"] == 0:
            assert c.analyze(0, case["sm_count"], case["t_min"]) == case["analyze"], case["name"]
            # the restatement names entities by local index; the golden by node id
            assert helpers.normalise_scheme(c.scheme(0, case["sm_count"], case["t_min"])) == \
                helpers.normalise_scheme(helpers.rename_scheme(case["scheme"], helpers.id_to_rank(case))), case["name"]


def test_appendix_a_goldens(orc):
    """SURVEY.md Appendix A, hand-derived from the code, as pinned by the reference run."""
    by = {(c["name"], c["sm_count"]): c for c in helpers.fixtures()}
    a1 = by[("fig2", 6)]["analyze"]
    assert (a1["proposed"], a1["greedy"], a1["graham_para"], a1["lower"]) == ("5", "7", "6", "4")
    a2 = by[("fig2", 8)]["scheme"]
    # entities are named by node id (Fig. 2's ids are 1..7): node 2 is split
    assert [s["parallel"] for s in a2["segmentations"]] == ["2:p1"]
    assert by[("fig2", 148)]["analyze"]["proposed"] == "4"
    a4 = by[("c1_fan_8_20_1", 148)]["analyze"]
    assert (a4["proposed"], a4["graham_para"], a4["lower"]) == ("28/9", "603/148", "3")
    assert by[("diamond_1_5_2_1", 4)]["analyze"]["proposed"] == "17/4"
    g = [sorted(int(m["entity"]) for m in grp["members"]) for grp in by[("c1_fan_8_20_1", 148)]["scheme"]["groups"]]
    assert g == [[0], list(range(1, 9)), [9]]
    quotas = [m["parallelism"] for m in by[("c1_fan_8_20_1", 148)]["scheme"]["groups"][1]["members"]]
    assert quotas == [19, 19, 19, 19, 18, 18, 18, 18]


@pytest.mark.parametrize("name,tag", [("corpus_default.npz", "default"), ("corpus_variants.npz", "heavy"),
                                      ("corpus_variants.npz", "fractional"), ("corpus_variants.npz", "wide")])
def test_corpus_bounds(orc, name, tag):
    b, res, cfg = helpers.corpus(name, tag)
    gen = orc.generate(b.n_dags, **cfg).pack()
    for k in ("node_off", "edge_off", "load_num", "load_den", "edges"):
        assert np.array_equal(getattr(gen, k), getattr(b, k)), k  # generator parity
    c = orc.corpus(b)
    for M, (st_ref, b_ref) in res.items():
        st, bounds, _ = c.evaluate(M)
        assert np.array_equal(st, st_ref)
        assert np.array_equal(bounds, b_ref), M


def test_scheme_goldens(orc):
    b, _, cfg = helpers.corpus()
    c = orc.corpus(b)
    n = 0
    for rec in helpers.schemes():
        assert helpers.normalise_scheme(c.scheme(rec["dag"], rec["sm_count"])) == \
            helpers.normalise_scheme(rec["scheme"])
        n += 1
    assert n == 360


@pytest.mark.skipif(not bindings.available("ref"), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("cfg", [dict(seed=9001), dict(seed=77, avg_load=120, max_width=12),
                                 dict(seed=5, integer_loads=False, avg_load=3, t_min="1/2")])
def test_restatement_vs_reference_library(orc, cfg):
    ref = bindings.Checker("ref")
    a, o = ref.generate(400, **cfg), orc.generate(400, **cfg)
    pa, po = a.pack(), o.pack()
    assert np.array_equal(pa.load_num, po.load_num) and np.array_equal(pa.edges, po.edges)
    tmin = cfg.get("t_min", 1)
    for M in (3, 16, 148):
        sa, ba, _ = a.evaluate(M, tmin)
        so, bo, _ = o.evaluate(M, tmin)
        assert np.array_equal(sa, so) and np.array_equal(ba, bo)
        for d in range(0, 400, 40):
            assert a.scheme(d, M, tmin) == o.scheme(d, M, tmin)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(bindings.LIBS["ref"]), "ref_test_dag_model")),
                    reason="reference test binaries not built")
@pytest.mark.parametrize("binary", ["ref_test_dag_model", "ref_test_exec_model"])
def test_reference_unit_tests(binary):
    """The reference's own doctest files (proj/tests/test_dag_model.cpp,
    test_exec_model.cpp) compiled against the shimmed reference library."""
    exe = os.path.join(os.path.dirname(bindings.LIBS["ref"]), binary)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout


@pytest.mark.skipif(not bindings.available("ref"), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed,tmin", [(1, 1), (2, "1/2"), (3, "3/2")])
def test_restatement_vs_reference_on_random_general_dags(orc, seed, tmin):
    """Fuzz: non-layered DAGs, shuffled ids, fractional and oversized loads."""
    from fractions import Fraction
    from paper_2602_20826_b200.batch import from_arrays, pack
    from tests import fuzz_dags
    b = pack(fuzz_dags.corpus(seed, 300, max_n=120, tmin=Fraction(tmin)))
    raw = from_arrays(b.node_off, b.edge_off, b.load_num, b.load_den, b.edges)
    ref = bindings.Checker("ref")
    a, o = ref.corpus(raw, min_load=Fraction(tmin)), orc.corpus(raw, min_load=Fraction(tmin))
    for M in (1, 3, 8, 37, 148):
        sa, ba, _ = a.evaluate(M, tmin)
        so, bo, _ = o.evaluate(M, tmin)
        assert np.array_equal(sa, so) and np.array_equal(ba, bo), M
        for d in range(0, 300, 15):
            if sa[d] == 0:
                assert a.scheme(d, M, tmin) == o.scheme(d, M, tmin), (M, d)


@pytest.mark.skipif(not bindings.available("ref"), reason="oracle/_ref not built (needs /root/reference)")
def test_paper_benchmark_families_vs_reference(orc):
    """Tables 1-2 DAG families (Gaussian elimination, Laplace, Stencil): the
    restatement's bounds and schemes equal the reference library's."""
    from paper_2602_20826_b200 import workloads
    from paper_2602_20826_b200.batch import from_arrays, pack
    dags = [d for avg in (4, 20) for d in workloads.paper_benchmarks(avg).values()]
    b = pack(dags)
    assert (b.pack_status == 0).all()
    raw = from_arrays(b.node_off, b.edge_off, b.load_num, b.load_den, b.edges)
    a, o = bindings.Checker("ref").corpus(raw), orc.corpus(raw)
    for M in (8, 30, 32, 148):
        sa, ba, _ = a.evaluate(M)
        so, bo, _ = o.evaluate(M)
        assert (sa == 0).all() and np.array_equal(sa, so) and np.array_equal(ba, bo), M
        for d in range(len(dags)):
            assert a.scheme(d, M) == o.scheme(d, M), (M, d)

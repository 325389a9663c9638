"""GPU fuzz parity: random general DAGs (shuffled ids, n up to 200, fractional
loads, oversized kernels, small M so Rule 1 truncates and nodes are split and
re-split) through K1 vs the restated oracle and, where built, the reference
itself (oracle/_ref); schedules vs the reference's write_scheme JSON."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import bindings
from paper_2602_20826_b200 import _lib, scheme
from paper_2602_20826_b200.batch import pack
from tests import fuzz_dags, helpers

pytestmark = pytest.mark.gpu


def _checkers():
    out = [bindings.Checker("oracle")]
    if bindings.available("ref"):
        out.append(bindings.Checker("ref"))
    return out


@pytest.mark.parametrize("seed,tmin,max_n", [(1, 1, 96), (2, Fraction(1, 2), 96), (3, 1, 200),
                                             (4, Fraction(3, 2), 60)])
def test_fuzz_bounds(seed, tmin, max_n):
    dags = fuzz_dags.corpus(seed, 600, max_n=max_n, tmin=Fraction(tmin))
    b = pack(dags)
    for M in (1, 2, 3, 5, 8, 16, 37, 148, 1000):
        st, bounds, _ = _lib.analyze(b, M, tmin)
        for chk in _checkers():
            c = chk.corpus(helpers_raw(b), min_load=tmin)
            st_o, b_o, _ = c.evaluate(M, tmin)
            assert np.array_equal(st, st_o), (chk.kind, M, np.nonzero(st != st_o)[0][:5])
            bad = np.nonzero((bounds != b_o).any(1))[0]
            assert len(bad) == 0, (chk.kind, M, bad[:5])


@pytest.mark.parametrize("seed,n_lo,n_hi,scale,Ms", [
    (31, 257, 700, 1, (2, 37, 148)),          # big classes, shuffled ids, fractional loads
    (32, 600, 1024, 1, (8, 148)),             # W = 16 class up to the limit
    (33, 2, 60, 1 << 20, (1, 3, 148)),        # wide values: 64/128-bit tiers, 128-bit overflow
    (34, 257, 400, 3, (5, 148)),              # scaled fractional loads in the big classes
])
def test_fuzz_big_and_wide(seed, n_lo, n_hi, scale, Ms):
    dags = fuzz_dags.corpus_sized(seed, 40, n_lo, n_hi, scale=scale)
    b = pack(dags)
    chk = bindings.Checker("ref" if bindings.available("ref") else "oracle")
    c = chk.corpus(helpers_raw(b))
    for M in Ms:
        st, bounds, _ = _lib.analyze(b, M)
        st_o, b_o, _ = c.evaluate(M, parallel=False)  # (an overflow inside the reference's OpenMP loop aborts it)
        assert np.array_equal(st, st_o), (M, np.nonzero(st != st_o)[0][:5], st[st != st_o][:5], st_o[st != st_o][:5])
        bad = np.nonzero((bounds != b_o).any(1))[0]
        assert len(bad) == 0, (M, bad[:5])
    if scale > 1:
        assert (st == 0).any()  # the tiers carry most DAGs


def test_fuzz_invalid_statuses():
    dags = fuzz_dags.broken(7, 200)
    b = pack(dags)
    st, bounds, _ = _lib.analyze(b, 8)
    ref =bindings.Checker("ref" if bindings.available("ref") else "oracle")
    for i, (nodes, edges) in enumerate(dags):
        one = helpers.fixture_raw_batch({"nodes": [[v, str(Fraction(l))] for v, l in nodes], "edges": edges})
        c = ref.corpus(one)
        s_ref, _, _ = c.evaluate(8)
        assert int(st[i]) == int(s_ref[0]), (i, int(st[i]), int(s_ref[0]))
    assert (st != 0).sum() >= 150


@pytest.mark.skipif(not bindings.available("ref"), reason="needs oracle/_ref")
@pytest.mark.parametrize("M", [3, 8, 148])
def test_fuzz_schemes_vs_reference(M):
    dags = fuzz_dags.corpus(11, 150, max_n=80)
    b = pack(dags)
    schemes, st = scheme.schedule_batch(b, M)
    # the tasks keep their (sparse, shuffled) node ids on both sides
    ref = bindings.Checker("ref").corpus_with_ids(helpers_raw(b), np.concatenate([np.asarray(i) for i in b.node_ids]))
    for d in range(len(dags)):
        if st[d] != 0:
            continue
        got = scheme.to_reference_json(schemes[d])
        assert helpers.normalise_scheme(got) == helpers.normalise_scheme(ref.scheme(d, M)), d


@pytest.mark.skipif(not bindings.available("ref"), reason="needs oracle/_ref")
@pytest.mark.parametrize("M", [8, 148])
def test_fuzz_big_schemes_vs_reference(M):
    """write_scheme JSON of big DAGs (k1_big in detail mode: variable-width
    unlaunched masks) with sparse, shuffled node ids on both sides."""
    dags = fuzz_dags.corpus_sized(41, 6, 257, 600)
    b = pack(dags)
    schemes, st = scheme.schedule_batch(b, M)
    ref = bindings.Checker("ref").corpus_with_ids(helpers_raw(b), np.concatenate([np.asarray(i) for i in b.node_ids]))
    st_r, _, _ = ref.evaluate(M, parallel=False)
    assert np.array_equal(st, st_r)
    assert (st == 0).sum() >= 3
    for d in range(len(dags)):
        if st[d] != 0:
            continue
        got = scheme.to_reference_json(schemes[d])
        assert helpers.normalise_scheme(got) == helpers.normalise_scheme(ref.scheme(d, M)), d


def helpers_raw(b):
    """The packed batch as the checkers take it (same arrays, id-free)."""
    from paper_2602_20826_b200.batch import from_arrays
    return from_arrays(b.node_off, b.edge_off, b.load_num, b.load_den, b.edges)


@pytest.mark.parametrize("seed", [21, 22])
def test_fuzz_compact16_matches_wide(seed):
    """Integer-load fuzz DAGs (shuffled ids, n up to 200, oversized loads)
    through the 16-bit wire form: same statuses and bounds as the wide form,
    which the oracle pins above."""
    dags = fuzz_dags.corpus(seed, 600, max_n=200)
    dags = [(nodes, edges) for nodes, edges in dags
            if all(Fraction(l).denominator == 1 and 1 <= Fraction(l) <= 0xFFFF for _, l in nodes)]
    assert len(dags) > 100
    b = pack(dags)
    assert b.compact16_ok()
    for M in (3, 8, 148):
        st, bounds, ng = _lib.analyze(b, M)
        st16, bounds16, ng16 = _lib.analyze16(b, M)
        assert np.array_equal(st, st16) and np.array_equal(bounds, bounds16) and np.array_equal(ng, ng16), M

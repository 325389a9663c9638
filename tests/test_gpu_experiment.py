"""Sweep driver (run_experiment / write_csv, experiment.cpp:81-161) over the
GPU batch boundary: byte-identical CSV with the reference's own driver
(tests/golden/experiments.json), and completion where the reference's
128-bit exact mean overflows."""
import json
import os
from fractions import Fraction

import pytest

from paper_2602_20826_b200 import experiment
from tests import helpers

pytestmark = pytest.mark.gpu


def _cases():
    with open(os.path.join(helpers.GOLDEN, "experiments.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['sweep']}{c['values']}_n{c['corpus_size']}")
def test_csv_matches_reference(case):
    rows = experiment.run_experiment(case["sweep"], case["values"], case["config"], case["sm_count"],
                                     case["corpus_size"])
    assert experiment.write_csv(rows) == case["csv"]


def test_large_sweep_completes_where_reference_overflows():
    rows = experiment.run_experiment("M", [4, 32, 148], dict(seed=1), 32, 1000)
    csv = experiment.write_csv(rows)
    ref_rows = [r for r in rows if r["method"] == "greedy_unaware"]
    assert all(r["mean_norm"] == 1 for r in ref_rows)
    prop = [r for r in rows if r["method"] == "proposed"]
    assert all(0 < r["mean_norm"] <= 1 for r in prop)  # Fig. 4: proposed <= greedy_unaware
    assert csv.count("\n") == 1 + 3 * 4


def test_format_fixed_matches_reference_semantics():
    f = experiment.format_fixed
    assert f(Fraction(1, 3), 6) == "0.333333"
    assert f(Fraction(2, 3), 6) == "0.666667"
    assert f(Fraction(-1, 8), 2) == "-0.13"   # half away from zero
    assert f(Fraction(5, 2), 0) == "3"
    assert f(Fraction(0), 3) == "0.000"

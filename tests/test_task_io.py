"""Task / trace I/O against the reference's read_task / write_task
(task_io.cpp:16-157), goldens made by oracle/_ref (tests/golden/sim.json)."""
import json
import os
from fractions import Fraction

import pytest

from paper_2602_20826_b200 import task_io, workloads
from paper_2602_20826_b200._lib import DagschedError
from paper_2602_20826_b200.simulator import SimEvent, SimTrace
from tests import helpers


def _golden():
    with open(os.path.join(helpers.GOLDEN, "sim.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _golden()["task_io"], ids=lambda c: c["doc"][:40])
def test_read_write_task_matches_reference(case):
    try:
        t = task_io.read_task(case["doc"], Fraction(case["min_load"]))
    except DagschedError as e:
        assert case["status"] != 0 and e.code == case["status"], (e, case["status"])
        return
    assert case["status"] == 0
    got = task_io.write_task(t, case["seed"])
    # the oracle's nlohmann copy prints integer arrays inline; compare documents
    assert json.loads(got) == json.loads(case["written"])
    assert got.endswith("}\n")


def test_write_task_layout_is_nlohmann_dump2():
    t = task_io.make_task([(1, 1), (2, "15/2")], [(1, 2)], period="10")
    assert task_io.write_task(t, seed=3) == (
        '{\n  "edges": [\n    [\n      1,\n      2\n    ]\n  ],\n  "nodes": [\n    {\n      "id": 1,\n'
        '      "load": "1"\n    },\n    {\n      "id": 2,\n      "load": "15/2"\n    }\n  ],\n'
        '  "period": "10",\n  "seed": 3\n}\n')


def test_task_file_round_trip(tmp_path):
    nodes, edges = workloads.make_example_task()
    t = task_io.make_task(nodes, edges)
    p = tmp_path / "fig2.json"
    task_io.write_task_file(t, str(p), seed=5)
    back = task_io.read_task_file(str(p))
    assert back.nodes == t.nodes and back.edges == t.edges and back.period is None
    with pytest.raises(DagschedError):
        task_io.read_task_file(str(tmp_path / "missing.json"))


@pytest.mark.parametrize("x,want", [(0.0, "0"), (1.0, "1"), (7.5, "7.5"), (0.1, "0.1"), (0.0001, "1e-04"),
                                    (0.001, "0.001"), (1e-05, "1e-05"), (1e20, "1e+20"), (1e15, "1e+15"), (123456789.0, "123456789"),
                                    (1e21, "1e+21"), (123456.789, "123456.789"), (2.5e-07, "2.5e-07"),
                                    (1.4151560559444937e+19, "14151560559444936704"), (-2.5, "-2.5")])
def test_to_chars_shortest(x, want):
    # values checked against libstdc++ std::to_chars(double) (GCC 13)
    assert task_io.to_chars_shortest(x) == want


@pytest.mark.parametrize("text,want", [("7.5", Fraction(15, 2)), ("15/2", Fraction(15, 2)), ("-3", Fraction(-3)),
                                       ("+0.25", Fraction(1, 4)), (".5", Fraction(1, 2)), ("5.", None),
                                       ("1e5", None), ("1/0", None), ("", None), ("-", None), (" 1", None),
                                       ("1/-2", None)])
def test_parse_rational(text, want):
    assert task_io.parse_rational(text) == want


def test_write_trace_format():
    tr = SimTrace([SimEvent("1", Fraction(0), Fraction(3, 2), 4), SimEvent("2:p1", Fraction(3, 2), Fraction(2), 2)],
                  Fraction(2))
    assert task_io.write_trace(tr) == "entity,start,finish,sms\n1,0,3/2,4\n2:p1,3/2,2,2\nmakespan,2,,\n"

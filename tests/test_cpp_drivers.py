"""§8(f) drivers through the kept C++ API against the reference's own code.

tests/cpp/drivers_dump.cpp builds twice from one source: against the
reference's headers and library (oracle/_ref/ref_drivers_dump, CPU) and
against include/dagsched + libdagsched_cpp.so (api_drivers_dump: K1 schedules
and bounds, K4 validation, K6 greedy simulation on the GPU). Their outputs —
task files, schedules, traces, CSVs, validation summaries as exact double bit
patterns, error classes and messages — must be identical.

One normalisation: oracle/_ref links the nlohmann/json copy shipped with
cudnn_frontend, which is patched ("Custom from FE") to print arrays of
integers on one line; the reference's stock nlohmann (and this API) print
one element per line. Integer arrays are collapsed on both sides before
comparing; everything else is byte for byte.
"""
import os
import re
import subprocess
from fractions import Fraction

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2602_20826_b200", "_lib")
REF = os.path.join(ROOT, "oracle", "_ref")
FIX = os.path.join(ROOT, "tests", "golden", "bench_fixtures")
API_BIN = os.path.join(LIB, "api_drivers_dump")
REF_BIN = os.path.join(REF, "ref_drivers_dump")

need_ref = pytest.mark.skipif(not os.path.exists(REF_BIN), reason="oracle/_ref not built")


def canon(text: str) -> str:
    return re.sub(r"\[\s*(-?\d+(?:,\s*-?\d+)*)\s*\]",
                  lambda m: "[" + ",".join(x.strip() for x in m.group(1).split(",")) + "]", text)


def run(binary, *args):
    r = subprocess.run([binary, FIX, *args], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    return r.stdout


@need_ref
def test_task_io_host_parts_match_reference():
    """read_task (exact strings, integers, JSON floats through to_chars, every
    validation error) and write_task, no device involved."""
    api, ref = run(API_BIN, "--host-only"), run(REF_BIN, "--host-only")
    assert '"load": "15/2"' in api and "unrepresentable number" in api
    assert canon(api) == canon(ref)


@need_ref
@pytest.mark.gpu
def test_drivers_match_reference():
    """write_scheme / simulate_scheme / simulate_greedy / write_trace /
    run_experiment / write_csv / run_validation / run_benchmarks /
    write_bench_table, section by section."""
    api, ref = canon(run(API_BIN)), canon(run(REF_BIN))
    sa = [s for s in api.split("== ") if s]
    sr = [s for s in ref.split("== ") if s]
    assert [s.splitlines()[0] for s in sa] == [s.splitlines()[0] for s in sr]
    for a, r in zip(sa, sr):
        if a != r:  # name the first differing line
            la, lr = a.splitlines(), r.splitlines()
            i = next((k for k in range(min(len(la), len(lr))) if la[k] != lr[k]), min(len(la), len(lr)))
            raise AssertionError(f"section {la[0]!r}, line {i}: {la[i] if i < len(la) else None!r} "
                                 f"!= {lr[i] if i < len(lr) else None!r}")


@pytest.mark.gpu
def test_run_experiment_completes_where_reference_overflows():
    """At 300 DAGs per point the reference's 128-bit running sum overflows
    (std::overflow_error); the kept API sums exactly in unbounded integers
    (means that do not fit 128 bits are truncated to a multiple of 10^-18,
    which cannot change a 6-digit half-away rounding) and its CSV equals the
    Python driver's, whose means are unbounded Fractions."""
    from paper_2602_20826_b200 import experiment
    api = run(API_BIN, "--experiment", "300")
    assert "overflow_error" not in api
    rows = experiment.run_experiment("M", [4, 8, 32, 148], {}, 148, 300)
    assert api == experiment.write_csv(rows)
    if os.path.exists(REF_BIN):
        assert "sweep M: overflow_error" in run(REF_BIN, "--experiment", "300")

"""Golden vectors for the simulator, task I/O and run_benchmarks, made by the
REFERENCE's own code (oracle/_ref: simulate_greedy, simulate_scheme +
check_precedence, write_trace, read_task/write_task, run_benchmarks +
write_bench_table). Writes tests/golden/sim.json.

Run from the repo root:  python tests/golden/make_golden_sim.py
"""
from __future__ import annotations

import glob
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import bindings as B  # noqa: E402
from paper_2602_20826_b200 import workloads  # noqa: E402
from paper_2602_20826_b200.batch import pack  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

TASK_DOCS = [
    '{"nodes": [{"id": 3, "load": 7.5}, {"id": 1, "load": "15/2"}], "edges": [[1, 3]], "period": "100"}',
    '{"nodes": [{"id": 0, "load": 2}, {"id": 1, "load": 0.5}, {"id": 2, "load": "1.25"}], '
    '"edges": [[0, 1], [0, 2], [0, 1]]}',
    '{"nodes": [{"id": 0, "load": 0.1}, {"id": 1, "load": 3}], "edges": [[0, 1]]}',
    '{"nodes": [{"id": 0, "load": 0.0001}, {"id": 1, "load": 2}], "edges": [[0, 1]]}',
    '{"nodes": [{"id": 0, "load": 1e-5}, {"id": 1, "load": 2}], "edges": [[0, 1]]}',
    '{"nodes": [{"id": 0, "load": 1e22}, {"id": 1, "load": 2}], "edges": [[0, 1]]}',
    '{"nodes": [{"id": 0, "load": 123456.789}, {"id": 1, "load": 2}], "edges": [[0, 1]], "period": 12.5}',
    '{"nodes": [{"id": 0, "load": "7.5x"}], "edges": []}',
    '{"nodes": [{"id": 0, "load": true}], "edges": []}',
    '{"nodes": [{"id": 0, "load": "3"}], "edges": [[0]]}',
    '{"nodes": [{"id": 0, "load": "3"}]}',
    '{"nodes": [], "edges": []}',
    '{"nodes": [{"id": 1, "load": 1}, {"id": 1, "load": 2}], "edges": []}',
    '{"nodes": [{"id": 1, "load": "1/2"}], "edges": []}',
    '{"nodes": [{"id": 1, "load": 2}, {"id": 2, "load": 2}], "edges": [[1, 2], [2, 1]]}',
    '{"nodes": [{"id": 1, "load": 2}, {"id": 2, "load": 2}], "edges": [[1, 9]]}',
    '{"nodes": [{"id": 1, "load": 2}, {"id": 2, "load": 2}, {"id": 3, "load": 1}], "edges": [[1, 3], [2, 3]]}',
    '{"nodes": [{"id": 1, "load": 2}], "edges": [], "period": "0"}',
    '{"nodes": [{"id": 1, "load": 2}], "edges": [], "period": -3}',
    'not json',
]


def main():
    out = {"generated_by": "oracle/_ref (reference sources + oracle/shim)"}
    # --- task I/O round trips (read_task -> write_task), incl. failures
    tio = []
    for k, doc in enumerate(TASK_DOCS):
        seed = 11 if k % 3 == 0 else None
        st, text = B.ref_task_roundtrip(doc, 1 if k != 2 else "1/10", seed)
        tio.append({"doc": doc, "min_load": "1" if k != 2 else "1/10", "seed": seed, "status": st,
                    "written": text})
    out["task_io"] = tio

    # --- simulate_greedy makespans over generated corpora
    chk = B.Checker("ref")
    greedy = []
    for cfg, n, M, runs, policy, scaled, smin, smax in (
            (dict(seed=1), 200, 148, 6, "random", False, 1, 1),
            (dict(seed=1), 200, 8, 6, "random", False, 1, 1),
            (dict(seed=2), 200, 32, 4, "fifo", False, 1, 1),
            (dict(seed=3, avg_load=200), 100, 148, 4, "random", True, "1/2", "1"),
            (dict(seed=4, integer_loads=False, avg_load=5), 100, 16, 4, "random", True, "1/3", "3/4"),
            (dict(seed=5, depth_min=10, depth_max=14, max_width=8), 60, 32, 3, "random", False, 1, 1)):
        corp = chk.generate(n, **cfg)
        st, mk = B.ref_sim_greedy(corp, M, runs, policy, 1000, scaled, 77, smin, smax)
        pb = corp.pack()
        greedy.append({"config": cfg, "n": n, "sm_count": M, "runs": runs, "policy": policy, "policy_seed": 1000,
                       "scaled": scaled, "time_seed": 77, "scale_min": str(smin), "scale_max": str(smax),
                       "status": st.tolist(), "makespan": mk.tolist(),
                       "traces": [B.ref_sim_greedy_trace(corp, d, M, policy, 1000 + 1, scaled, 77, smin, smax)
                                  for d in range(3)],
                       "n_nodes": int(pb.node_off[-1])})
    out["greedy"] = greedy

    # --- simulate_scheme traces (+ check_precedence) on hand-built DAGs
    sch = []
    for name, dag, M, scaled, seed, smin, smax in (
            ("fig2", workloads.make_example_task(), 8, False, 0, 1, 1),
            ("fig2", workloads.make_example_task(), 6, True, 5, "1/2", "1"),
            ("c1", workloads.c1_fork_join(), 148, False, 0, 1, 1),
            ("c1", workloads.c1_fork_join(), 32, True, 9, "1/4", "3/4"),
            ("c3", workloads.inception_dag(), 32, True, 3, "1/2", "1"),
            ("c4", workloads.oversized_dag(0, 148), 148, False, 0, 1, 1)):
        corp = chk.corpus(pack([dag]))
        sch.append({"name": name, "sm_count": M, "scaled": scaled, "time_seed": seed, "scale_min": str(smin),
                    "scale_max": str(smax), "trace": B.ref_sim_scheme_trace(corp, 0, M, scaled, seed, smin, smax)})
    out["scheme_traces"] = sch

    # --- run_benchmarks + write_bench_table on the unit-load fixtures
    paths = sorted(glob.glob(os.path.join(OUT, "bench_fixtures", "*.json")))
    bench = []
    for sms, avgs, runs, seed in (([148, 32, 8], [1, 20, 200], 20, 1), ([16], [5], 50, 99)):
        csv = B.ref_run_benchmarks(paths, sms, avgs, runs, seed)
        bench.append({"fixtures": [os.path.basename(p) for p in paths], "sm_counts": sms, "avg_loads": avgs,
                      "greedy_runs": runs, "seed": seed, "csv": csv})
    out["benchmarks"] = bench
    with open(os.path.join(OUT, "sim.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(OUT, "sim.json"))


if __name__ == "__main__":
    main()

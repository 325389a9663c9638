"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

The reference's own sources (/root/reference/proj/src) are compiled against
oracle/shim into oracle/_ref/libdagsched_ref.so (``make -C oracle ref``); this
script drives that library through its public API (generate_corpus,
evaluate_corpus, lower_bound, schedule + write_scheme, analyze) and writes:

  fixtures.json            hand-built DAGs (paper Fig. 2, fan/C1, diamond,
                           chain, Inception/C3, oversized/C4, invalid DAGs,
                           fractional loads / t_min) with the reference's
                           status, analyze() report and write_scheme() JSON
  corpus_default.npz       generate_corpus(GenConfig{}, seed=1, 1000) packed,
                           with status + 5 bounds at M in {4, 8, 32, 148}
  corpus_variants.npz      three more generator configs (heavy loads,
                           fractional loads, wide/deep) at M in {8, 32, 148}
  schemes.jsonl.gz         write_scheme() JSON for the first 120 DAGs of
                           corpus_default at M in {8, 32, 148}

Run from the repo root:  python tests/golden/make_golden.py
Only this container has /root/reference; the GPU box uses the committed files.
"""
from __future__ import annotations

import gzip
import json
import os
import sys
from fractions import Fraction

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bindings import Checker  # noqa: E402
from paper_2602_20826_b200 import workloads  # noqa: E402
from paper_2602_20826_b200.batch import from_arrays  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def raw_pack(dags):
    """Pack without validation: ids are mapped to ranks; an endpoint that is
    not a node id maps to index n (out of range) so the reference sees an
    unknown node exactly as DagTask::make would (dag.cpp:57-60)."""
    node_off, edge_off, nums, dens, words = [0], [0], [], [], []
    for nodes, edges in dags:
        nodes = sorted(((int(i), Fraction(l)) for i, l in nodes), key=lambda t: t[0])
        ids = [i for i, _ in nodes]
        idx = {i: k for k, i in enumerate(ids)}
        for _, l in nodes:
            nums.append(l.numerator)
            dens.append(l.denominator)
        for u, v in edges:
            words.append((idx.get(u, len(ids)) << 16) | idx.get(v, len(ids)))
        node_off.append(len(nums))
        edge_off.append(len(words))
    return from_arrays(node_off, edge_off, nums, dens, words)


def fixtures():
    F = []
    ex = workloads.make_example_task()
    for M in (3, 4, 5, 6, 8, 32, 148):
        F.append(("fig2", ex, M, 1))
    F.append(("fig2_tmin_half", ex, 8, "1/2"))
    F.append(("c1_fan_8_20_1", workloads.c1_fork_join(), 148, 1))
    F.append(("c1_fan_8_20_1", workloads.c1_fork_join(), 32, 1))
    F.append(("fan_12_7_3", workloads.make_fan(12, 7, 3), 16, 1))
    F.append(("diamond_1_5_2_1", workloads.make_diamond(1, 5, 2, 1), 4, 1))
    F.append(("diamond_unit", workloads.make_diamond(), 4, 1))
    F.append(("chain_4_4", workloads.make_chain([4, 4]), 4, 1))
    F.append(("chain_mixed", workloads.make_chain([1, 30, 2, 300, 7]), 148, 1))
    F.append(("single_node", ([(0, 5)], []), 4, 1))
    F.append(("single_node_big", ([(0, 1000)], []), 148, 1))
    F.append(("fractional", ([(0, "3/2"), (1, "15/2"), (2, "7/3"), (3, 1)],
                             [(0, 1), (0, 2), (1, 3), (2, 3)]), 8, 1))
    F.append(("fractional_tmin", ([(0, "3/2"), (1, "15/2"), (2, "7/3"), (3, "1/2")],
                                  [(0, 1), (0, 2), (1, 3), (2, 3)]), 16, "1/2"))
    for M in (32, 148):
        F.append(("c3_inception", workloads.inception_dag(), M, 1))
    for s in range(3):
        for M in (32, 148):
            F.append((f"c4_oversized_{s}", workloads.oversized_dag(s, M), M, 1))
    # invalid DAGs (dag.cpp:22-138)
    F.append(("cycle", ([(1, 1), (2, 1)], [(1, 2), (2, 1)]), 4, 1))
    F.append(("cycle3", ([(0, 1), (1, 1), (2, 1), (3, 1)], [(0, 1), (1, 2), (2, 1), (2, 3)]), 4, 1))
    F.append(("self_loop", ([(1, 1)], [(1, 1)]), 4, 1))
    F.append(("two_sources", ([(0, 1), (1, 1), (2, 1)], [(0, 2), (1, 2)]), 4, 1))
    F.append(("two_sinks", ([(0, 1), (1, 1), (2, 1)], [(0, 1), (0, 2)]), 4, 1))
    F.append(("load_below_min", ([(3, "1/2")], []), 4, 1))
    F.append(("unknown_endpoint", ([(0, 1)], [(0, 9)]), 4, 1))
    F.append(("duplicate_edges", ([(0, 1), (1, 2), (2, 1)], [(0, 1), (0, 1), (1, 2), (0, 2)]), 4, 1))
    # tasks made with DagTask::make's default floor (min_load = 1) on a
    # platform whose t_min is above some load: only schedule() refuses them
    # (scheduler.cpp:177-182); the other bounds exist (analysis.cpp:40-81)
    F.append(("load_below_tmin", ([(10, 1), (11, 5), (12, 2), (13, 3)], [(10, 11), (10, 12), (11, 13), (12, 13)]),
              8, 2, 1))
    F.append(("load_below_tmin_frac", ([(0, "3/2"), (1, 7), (2, 1)], [(0, 1), (1, 2)]), 4, "5/2", 1))
    return F


def main():
    ref = Checker("ref")
    cases = []
    for name, (nodes, edges), M, tmin, *minl in fixtures():
        b = raw_pack([(nodes, edges)])
        ids = sorted(int(i) for i, _ in nodes)
        min_load = Fraction(minl[0]) if minl else Fraction(tmin)
        # the tasks carry their real node ids, so write_scheme names entities by id
        c = ref.corpus_with_ids(b, ids, min_load=min_load)
        # serial: an exception inside the reference's OpenMP loop would terminate
        st, bounds, _ = c.evaluate(M, Fraction(tmin), parallel=False)
        case = {"name": name, "nodes": [[int(i), str(Fraction(l))] for i, l in nodes],
                "edges": [[int(u), int(v)] for u, v in edges], "sm_count": M,
                "t_min": str(Fraction(tmin)), "status": int(st[0]),
                "bounds": [int(x) for x in bounds[0]]}
        if minl:
            case["min_load"] = str(min_load)
            st2, b2, _ = c.evaluate(M, Fraction(tmin), mask=0x1E, parallel=False)  # every method but proposed
            case["status_no_proposed"] = int(st2[0])
            case["bounds_no_proposed"] = [int(x) for x in b2[0]]
        if st[0] == 0:
            case["analyze"] = c.analyze(0, M, Fraction(tmin))
            case["scheme"] = c.scheme(0, M, Fraction(tmin))
        cases.append(case)
    with open(os.path.join(OUT, "fixtures.json"), "w") as f:
        json.dump({"generated_by": "oracle/_ref (reference sources + oracle/shim)",
                   "cases": cases}, f, indent=1, sort_keys=True)

    def corpus_npz(path, configs, Ms, n):
        arrays = {}
        for tag, cfg in configs.items():
            corp = ref.generate(n, **cfg)
            pb = corp.pack()
            for k in ("node_off", "edge_off", "load_num", "load_den", "edges"):
                arrays[f"{tag}__{k}"] = getattr(pb, k)
            arrays[f"{tag}__config"] = np.frombuffer(json.dumps(cfg).encode(), np.uint8)
            for M in Ms:
                st, bounds, _ = corp.evaluate(M)
                arrays[f"{tag}__status_M{M}"] = st
                arrays[f"{tag}__bounds_M{M}"] = bounds
        np.savez_compressed(path, **arrays)

    corpus_npz(os.path.join(OUT, "corpus_default.npz"), {"default": dict(seed=1)},
               (4, 8, 32, 148), 1000)
    corpus_npz(os.path.join(OUT, "corpus_variants.npz"), {
        "heavy": dict(seed=100, avg_load=200),
        "fractional": dict(seed=200, integer_loads=False, avg_load=5),
        "wide": dict(seed=300, depth_min=6, depth_max=10, max_width=24, avg_load=40),
    }, (8, 32, 148), 250)

    corp = ref.generate(120, seed=1)
    with gzip.open(os.path.join(OUT, "schemes.jsonl.gz"), "wt") as f:
        for M in (8, 32, 148):
            for d in range(120):
                f.write(json.dumps({"dag": d, "sm_count": M, "scheme": corp.scheme(d, M)},
                                   sort_keys=True) + "\n")
    # run_validation (experiment.cpp:163-240): the reference's own summary
    from oracle.bindings import ref_run_validation
    vals = []
    for cfg, n, M, S, smin, smax in ((dict(seed=1), 300, 32, 10, "1/2", "1"),
                                     (dict(seed=5, avg_load=4), 200, 8, 10, "1/4", "3/4"),
                                     (dict(seed=9), 300, 148, 5, "9/10", "1"),
                                     (dict(seed=13, avg_load=200, max_width=12), 100, 148, 8, "1/3", "1"),
                                     (dict(seed=17, integer_loads=False, avg_load=5), 150, 16, 10, "1/2", "1")):
        r = ref_run_validation(n, M, S, smin, smax, **cfg)
        vals.append({"config": cfg, "corpus_size": n, "sm_count": M, "samples": S, "scale_min": smin,
                     "scale_max": smax, "summary": {k: (v.hex() if isinstance(v, float) else v)
                                                    for k, v in r.items()}})
    with open(os.path.join(OUT, "validation.json"), "w") as f:
        json.dump(vals, f, indent=1)
    # run_experiment + write_csv (experiment.cpp:81-161), at sizes where the
    # reference's 128-bit exact mean does not overflow
    from oracle.bindings import ref_run_experiment
    exps = []
    for sweep, values, M, n, cfg in (("M", [148], 148, 20, dict(seed=3)), ("M", [4, 8], 8, 20, dict(seed=3)),
                                     ("M", [148, 256], 148, 30, dict(seed=3)), ("P", [4, 6], 148, 15, dict(seed=3)),
                                     ("V", [3, 4], 148, 15, dict(seed=3, max_width=4))):
        exps.append({"sweep": sweep, "values": values, "sm_count": M, "corpus_size": n, "config": cfg,
                     "csv": ref_run_experiment(sweep, values, M, n, **cfg)})
    with open(os.path.join(OUT, "experiments.json"), "w") as f:
        json.dump(exps, f, indent=1)
    # build_blocks / local_paths / build_groups / scale_parallelism /
    # parallel_candidates: tests/cpp/division_dump.cpp against the reference
    import subprocess
    dump = os.path.join(os.path.dirname(OUT), "..", "oracle", "_ref", "ref_division_dump")
    text = subprocess.run([dump], capture_output=True, text=True, check=True).stdout
    with gzip.open(os.path.join(OUT, "division.json.gz"), "wt", compresslevel=9) as f:
        f.write(text)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()

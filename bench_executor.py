#!/usr/bin/env python
"""Executor benchmark (configs C1-C4): measured DAG makespan vs analysed bound.

For every DAG: K1 schedules it on the GPU (ds_schedule_batch, M = 148), K3
turns the schedule into one CUDA Graph of K2 node kernels (grid = SM quota,
one CTA per SM), and the graph is replayed R times; each replay's makespan is
first-CTA-start -> last-CTA-end on %globaltimer. Next to it, the same DAG runs
as a serial stream and as naive multi-stream launch (original edges only,
every kernel at min(m^max, M)).

Time unit: one load unit = ``--unit`` elements per SM of the node kernel.
tau = the time of one unit on every SM at once (148 CTAs x unit elements,
full HBM contention, CUDA events) — the worst case a kernel of the schedule
can see, since a group never holds more than 148 SMs. bound_us = bound x tau;
per-group graph dependency latency delta (a chain of minimal kernels) is
measured and reported separately (SURVEY.md §7 hard part 4).

Writes one JSON document (default profiles/r01_executor.json) and prints a
one-line summary.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2602_20826_b200 import _lib, scheme, workloads  # noqa: E402
from paper_2602_20826_b200 import executor as X  # noqa: E402
from paper_2602_20826_b200.batch import pack  # noqa: E402

M = 148


def stats(a):
    a = np.asarray(a, np.float64)
    return {"p50": float(np.percentile(a, 50)), "p99": float(np.percentile(a, 99)), "max": float(a.max()),
            "mean": float(a.mean()), "min": float(a.min())}


def calibrate(unit, workload, reps=50):
    ms, span = X.node_kernel_bench(workload, M, unit, reps=reps)
    return ms * 1e3, span / 1e3  # us per unit at full contention (events), globaltimer span


def chain_delta(n=64, reps=50):
    """Graph dependency latency: a chain of n 1-CTA minimal kernels."""
    loads = [1] * n
    edges = [(i, i + 1) for i in range(n - 1)]
    plan = X.plan_baseline("serial", loads, edges, M, 4)
    ex = X.Executor(plan)
    res = ex.run(reps, warmup=3, stamps=False)
    ex.close()
    return float(np.median(res.makespan_us)) / n


def dag_from_batch(b, d):
    n0, n1 = int(b.node_off[d]), int(b.node_off[d + 1])
    e0, e1 = int(b.edge_off[d]), int(b.edge_off[d + 1])
    loads = [int(x) if den == 1 else (int(x), int(den)) for x, den in zip(b.load_num[n0:n1], b.load_den[n0:n1])]
    edges = [(int(w) >> 16, int(w) & 0xFFFF) for w in b.edges[e0:e1]]
    return loads, edges


def run_dag(loads, edges, sch, unit, tau_us, replays, workload, check_every):
    out = {"n": len(loads), "groups": len(sch.groups), "segmentations": len(sch.segmentations),
           "launches": sum(len(g.launches) for g in sch.groups),
           "bound_units": str(sch.bounds["proposed"]), "greedy_units": str(sch.bounds["greedy"])}
    bound_us = float(sch.bounds["proposed"]) * tau_us
    out["bound_us"] = bound_us
    res = {}
    for kind in ("proposed", "serial", "multistream"):
        if kind == "proposed":
            plan = X.plan_from_scheme(sch, loads, unit, barrier_groups=True)
        else:
            plan = X.plan_baseline(kind, loads, edges, M, unit)
        ex = X.Executor(plan, workload=workload)
        r = ex.run(replays, warmup=3, stamps=True)
        viol_prec = viol_sm = viol_grp = 0
        for k in range(0, replays, check_every):
            viol_prec += len(X.check_precedence(plan, r, k))
            viol_sm += X.check_sm_exclusive(plan, r, k)
            viol_grp += X.group_overlap_violations(plan, r, k)
        ex.close()
        res[kind] = {"makespan_us": stats(r.makespan_us), "launch_us": stats(r.launch_ms * 1e3),
                     "precedence_violations": viol_prec, "sm_overlap_violations": viol_sm,
                     "group_order_violations": viol_grp, "checked_replays": len(range(0, replays, check_every))}
        if kind == "proposed":
            out["ratio_to_bound"] = stats(r.makespan_us / bound_us)
            out["over_bound_replays"] = int((r.makespan_us > bound_us).sum())
    out.update(res)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--replays", type=int, default=1000)
    ap.add_argument("--c2-dags", type=int, default=100)
    ap.add_argument("--unit", type=int, default=1 << 17, help="elements per load unit per SM")
    ap.add_argument("--workload", type=int, default=X.WL_MIX32)
    ap.add_argument("--check-every", type=int, default=25)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_executor.json"))
    args = ap.parse_args()

    t_start = time.time()
    doc = {"sm_count": M, "unit_elems": args.unit, "workload": args.workload,
           "bytes_per_elem": X.BYTES_PER_ELEM[args.workload], "replays": args.replays}
    tau_us, tau_span_us = calibrate(args.unit, args.workload)
    doc["tau_us"] = tau_us
    doc["tau_globaltimer_us"] = tau_span_us
    doc["delta_us_per_dependency"] = chain_delta()
    # node-kernel roofline: 148 CTAs x 4 Mi elements (4.6 GB traffic, >> L2)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    roof = {}
    for wl, name in ((X.WL_MIX32, "mix32_ldg128"), (X.WL_MIX32_BULK, "mix32_bulk_tma"), (X.WL_AXPY32, "axpy_fp32")):
        ms, _ = X.node_kernel_bench(wl, M, 1 << 22, reps=20)
        gbs = M * (1 << 22) * X.BYTES_PER_ELEM[wl] / (ms * 1e-3) / 1e9
        roof[name] = {"ms": ms, "GB/s": gbs, "frac_of_measured_peak": gbs / peaks["hbm_gbs"]}
    doc["node_kernel_roofline"] = roof
    doc["hbm_peak_gbs"] = peaks["hbm_gbs"]

    cases = []
    cfgs = args.configs.split(",")
    if "c1" in cfgs:
        cases.append(("c1_fan_8_20_1", workloads.c1_fork_join()))
    if "c3" in cfgs:
        cases.append(("c3_inception", workloads.inception_dag()))
    if "c4" in cfgs:
        for s in range(3):
            cases.append((f"c4_oversized_{s}", workloads.oversized_dag(s, M)))
    if "c2" in cfgs:
        corpus = _lib.Corpus(600, seed=1)
        b = corpus.batch()
        sizes = np.diff(b.node_off.astype(np.int64))
        picked = [d for d in range(b.n_dags) if 20 <= sizes[d] <= 50][:args.c2_dags]
        for d in picked:
            cases.append((f"c2_seed{1 + d}", dag_from_batch(b, d)))
    # schedule everything on the GPU in one batch
    packed = []
    for name, (nodes, edges) in cases:
        packed.append((nodes, edges))
    batch = pack(packed)
    schemes, st = scheme.schedule_batch(batch, M)
    results = []
    for (name, (nodes, edges)), sch, s in zip(cases, schemes, st):
        if s != 0:
            results.append({"name": name, "status": int(s)})
            continue
        nodes = list(nodes)
        if nodes and isinstance(nodes[0], tuple):
            nodes = sorted(nodes, key=lambda t: t[0])
            ids = [i for i, _ in nodes]
            idx = {i: k for k, i in enumerate(ids)}
            loads = [l for _, l in nodes]
            edges = [(idx[u], idx[v]) for u, v in edges]
        else:
            loads = nodes
        r = run_dag(loads, edges, sch, args.unit, tau_us, args.replays, args.workload, args.check_every)
        r["name"] = name
        results.append(r)
        print(f"{name}: n={r['n']} groups={r['groups']} bound={r['bound_units']}u={r['bound_us']:.1f}us "
              f"proposed p50={r['proposed']['makespan_us']['p50']:.1f} max={r['proposed']['makespan_us']['max']:.1f} "
              f"serial p50={r['serial']['makespan_us']['p50']:.1f} multi p50={r['multistream']['makespan_us']['p50']:.1f} "
              f"over={r['over_bound_replays']}", flush=True)
    doc["dags"] = results
    ok = [r for r in results if "proposed" in r]

    def agg(prefix):
        sel = [r for r in ok if r["name"].startswith(prefix)]
        if not sel:
            return None
        return {
            "dags": len(sel),
            "replays_over_bound": int(sum(r["over_bound_replays"] for r in sel)),
            "max_ratio_to_bound": max(r["ratio_to_bound"]["max"] for r in sel),
            "median_ratio_to_bound": float(np.median([r["ratio_to_bound"]["p50"] for r in sel])),
            "proposed_p50_us_mean": float(np.mean([r["proposed"]["makespan_us"]["p50"] for r in sel])),
            "serial_p50_us_mean": float(np.mean([r["serial"]["makespan_us"]["p50"] for r in sel])),
            "multistream_p50_us_mean": float(np.mean([r["multistream"]["makespan_us"]["p50"] for r in sel])),
            "proposed_beats_multistream_p50": int(sum(r["proposed"]["makespan_us"]["p50"] <
                                                      r["multistream"]["makespan_us"]["p50"] for r in sel)),
            "proposed_beats_multistream_p99": int(sum(r["proposed"]["makespan_us"]["p99"] <
                                                      r["multistream"]["makespan_us"]["p99"] for r in sel)),
            "precedence_violations": int(sum(r[k]["precedence_violations"] for r in sel
                                             for k in ("proposed", "serial", "multistream"))),
            "sm_overlap_violations": int(sum(r[k]["sm_overlap_violations"] for r in sel
                                             for k in ("proposed", "serial", "multistream"))),
            "group_order_violations": int(sum(r["proposed"]["group_order_violations"] for r in sel)),
        }

    doc["summary"] = {k: agg(k) for k in ("c1", "c2", "c3", "c4")}
    doc["wall_s"] = time.time() - t_start
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({"tau_us": tau_us, "delta_us": doc["delta_us_per_dependency"],
                      "roofline": {k: round(v["frac_of_measured_peak"], 3) for k, v in roof.items()},
                      "summary": doc["summary"]}))


if __name__ == "__main__":
    main()
